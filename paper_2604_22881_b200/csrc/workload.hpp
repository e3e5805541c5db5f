// Trace generation (reference workload.cpp:85) shared by capi.cpp and workload.cpp.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/mtkv_b200.h"

namespace mtkv_b200 {
struct TraceRec {
  uint64_t ts;
  uint32_t user, dn, nc;
  std::vector<uint32_t> tokens, cands;
};
int generate(const mtkv_gen_config& g, std::vector<TraceRec>& out, std::string& err);
std::string to_jsonl(const std::vector<TraceRec>& tr);
}  // namespace mtkv_b200
