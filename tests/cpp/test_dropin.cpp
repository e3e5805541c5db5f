// Drop-in proof (TEST INFRASTRUCTURE): the reference's own engine / manager test
// cases, restated once as templates and run against BOTH the unmodified
// reference (mtkv::Engine<B>, mtkv::CacheManager from oracle/_ref/libmtkv_ref.so)
// and the B200 path through include/mtkv_b200_engine.hpp
// (mtkv::b200::Engine<B>, mtkv::b200::CacheManager over libmtkv_b200.so).
// Each case's assertions must hold for both, and the two implementations'
// observable results (RunReport::to_json, dump_page_map, plans, evictions,
// page ids) must be identical.
//
// Cases (reference file:line):
//   tests/test_sim.cpp:36   empty trace yields a zeroed report
//   tests/test_sim.cpp:47   resident prefix: second visit is a full device hit
//   tests/test_sim.cpp:58   unlimited capacity with chunk=page keeps total hit at 100%
//   tests/test_sim.cpp:75   two-user alternating eviction (hierarchical, gpu_only)
//   tests/test_sim.cpp:115  tokens processed across modes
//   tests/test_sim.cpp:139  gpu hit ratios agree between gpu_only and hierarchical
//   tests/test_sim.cpp:170  value backend: logits are mode-invariant
//                           (B200: bf16 storage / fp32 math, bars stated below)
//   tests/test_sim.cpp:230  report invariants and determinism
//   tests/test_manager.cpp:91-256  manager: first visit, resident prefix, same user
//                           twice, round-robin eviction, zero-copy eviction, locking
//                           protocol, oversized batches, batch members protected
//
// Built by oracle/Makefile (target dropin) into oracle/_ref/test_dropin against
// the reference headers; run by tests/test_dropin.py (manager cases on CPU,
// everything on the GPU with --engine).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <set>
#include <string>
#include <vector>

#include <mtkv/sim.hpp>

#include "mtkv_b200_engine.hpp"

using namespace mtkv;

namespace {

int g_checks = 0, g_failed = 0;
std::string g_case;

#define CHECK(...)                                                                      \
  do {                                                                                  \
    ++g_checks;                                                                         \
    if (!(__VA_ARGS__)) {                                                               \
      ++g_failed;                                                                       \
      std::printf("FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #__VA_ARGS__); \
    }                                                                                   \
  } while (0)
#define CHECK_FALSE(x) CHECK(!(x))
#define REQUIRE(x)                                                                     \
  do {                                                                                 \
    CHECK(x);                                                                          \
    if (!(x)) throw std::runtime_error("REQUIRE failed: " #x);                         \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                                       \
  do {                                                                                 \
    bool thrown_ = false;                                                              \
    try {                                                                              \
      expr;                                                                            \
    } catch (const T&) {                                                               \
      thrown_ = true;                                                                  \
    } catch (...) {                                                                    \
    }                                                                                  \
    CHECK(thrown_ && #expr " throws " #T);                                             \
  } while (0)

bool approx(double a, double b, double eps = 1e-12) { return std::fabs(a - b) <= eps * std::max(1.0, std::fabs(b)); }

Request treq(std::uint64_t ts, UserId u, std::uint32_t delta, std::uint32_t cands = 1) {
  Request r;
  r.timestamp = ts;
  r.user = u;
  r.new_token_count = delta;
  r.candidate_count = cands;
  return r;
}

KVConfig tiny_cfg() {
  KVConfig cfg;
  cfg.num_layers = 2;
  cfg.num_heads = 1;
  cfg.head_dim = 4;
  cfg.page_size = 32;
  cfg.chunk_size = 64;
  cfg.device_pages = 256;
  cfg.offload_quota = 512;
  return cfg;
}

template <class E>
std::string fingerprint(E& eng, const RunReport& r) {
  return r.to_json() + "|" + eng.dump_page_map();
}

// ------------------------------------------------------------ test_sim.cpp ---
using RefTag = mtkv::Engine<TagBackend>;
using B2Tag = mtkv::b200::Engine<TagBackend>;

template <class E>
std::string sim_empty() {
  EngineOptions opts;
  E eng(tiny_cfg(), CostModel{}, opts);
  RunReport r = eng.run({});
  CHECK(r.batches == 0);
  CHECK(r.tokens_processed == 0);
  for (double s : r.step_ms) CHECK(s == 0.0);
  CHECK(r.total_latency_ms == 0.0);
  CHECK(r.gpu_hit_ratio == 1.0);
  CHECK(r.total_hit_ratio == 1.0);
  return fingerprint(eng, r);
}

template <class E>
std::string sim_resident() {
  EngineOptions opts;
  E eng(tiny_cfg(), CostModel{}, opts);
  RunReport r = eng.run({treq(0, 1, 100), treq(1000, 1, 50)});
  CHECK(r.gpu_hit_ratio == 1.0);
  CHECK(r.total_hit_ratio == 1.0);
  CHECK(r.tokens_processed == 100 + 1 + 50 + 1);
  CHECK(r.evictions == 0);
  eng.check_conservation();
  return fingerprint(eng, r);
}

template <class E>
std::string sim_unlimited() {
  KVConfig cfg = tiny_cfg();
  cfg.chunk_size = cfg.page_size;
  cfg.device_pages = 4096;
  std::vector<Request> trace;
  std::uint64_t ts = 0;
  for (int round = 0; round < 4; ++round)
    for (UserId u = 0; u < 6; ++u) trace.push_back(treq(ts++, u, 70 + u));
  EngineOptions opts;
  E eng(cfg, CostModel{}, opts);
  RunReport r = eng.run(trace);
  CHECK(r.gpu_hit_ratio == 1.0);
  CHECK(r.total_hit_ratio == 1.0);
  CHECK(r.evictions == 0);
  eng.check_conservation();
  return fingerprint(eng, r);
}

template <class E>
std::string sim_alternating(Mode mode) {
  KVConfig cfg = tiny_cfg();
  cfg.device_pages = 9;
  cfg.offload_quota = 256;
  std::vector<Request> trace;
  std::uint64_t ts = 0;
  for (std::uint32_t delta : {192u, 32u, 32u}) {
    trace.push_back(treq(ts++, 1, delta));
    trace.push_back(treq(ts++, 2, delta));
  }
  EngineOptions opts;
  opts.mode = mode;
  E eng(cfg, CostModel{}, opts);
  RunReport r = eng.run(trace);
  CHECK(approx(r.gpu_hit_ratio, 0.0));
  CHECK(r.evictions == 5);
  if (mode == Mode::Hierarchical) {
    CHECK(approx(r.total_hit_ratio, 768.0 / 832.0));
    CHECK(r.tail_tokens_lost == 64);
    CHECK(eng.quota().in_flight == 0);
    CHECK(eng.manager().occupied_pages() + eng.device().free_count() == cfg.device_pages);
  } else {
    CHECK(approx(r.total_hit_ratio, 0.0));
  }
  eng.check_conservation();
  return fingerprint(eng, r);
}

template <class E>
std::string sim_tokens_across_modes() {
  KVConfig cfg = tiny_cfg();
  EngineOptions opts;
  std::string fp;
  for (Mode m : {Mode::Recompute, Mode::GpuOnly, Mode::Hierarchical}) {
    opts.mode = m;
    E eng(cfg, CostModel{}, opts);
    RunReport r = eng.run({treq(0, 1, 10, 2)});
    CHECK(r.tokens_processed == 12);
    fp += r.to_json();
  }
  std::vector<Request> trace = {treq(0, 1, 5), treq(1, 1, 5), treq(2, 1, 5)};
  opts.mode = Mode::Hierarchical;
  E reuse(cfg, CostModel{}, opts);
  RunReport a = reuse.run(trace);
  CHECK(a.tokens_processed == 3 * (5 + 1));
  opts.mode = Mode::Recompute;
  E re(cfg, CostModel{}, opts);
  RunReport b = re.run(trace);
  CHECK(b.tokens_processed == 6 + 11 + 16);
  return fp + a.to_json() + b.to_json();
}

template <class E>
std::string sim_hit_ratios_agree() {
  GenConfig g;
  g.num_users = 30;
  g.total_requests = 400;
  g.mean_final_len = 600;
  g.max_len = 2000;
  g.seed = 12;
  auto trace = generate_trace(g);
  KVConfig cfg = tiny_cfg();
  cfg.chunk_size = 128;
  cfg.device_pages = 300;
  cfg.offload_quota = 4096;
  EngineOptions opts;
  opts.mode = Mode::GpuOnly;
  opts.batch_size = 4;
  E gpu(cfg, CostModel{}, opts);
  RunReport rg = gpu.run(trace);
  opts.mode = Mode::Hierarchical;
  E hier(cfg, CostModel{}, opts);
  RunReport rh = hier.run(trace);
  CHECK(approx(rg.gpu_hit_ratio, rh.gpu_hit_ratio));
  CHECK(approx(rg.total_hit_ratio, rg.gpu_hit_ratio));
  CHECK(rh.total_hit_ratio >= rh.gpu_hit_ratio);
  CHECK(rh.total_latency_ms <= rg.total_latency_ms);
  hier.check_conservation();
  gpu.check_conservation();
  return fingerprint(gpu, rg) + fingerprint(hier, rh);
}

template <class E>
std::string sim_determinism() {
  GenConfig g;
  g.num_users = 20;
  g.total_requests = 200;
  g.mean_final_len = 400;
  g.max_len = 1500;
  g.seed = 3;
  auto trace = generate_trace(g);
  KVConfig cfg = tiny_cfg();
  cfg.device_pages = 200;
  EngineOptions opts;
  opts.batch_size = 4;
  opts.seed = 9;
  E e1(cfg, CostModel{}, opts);
  RunReport a = e1.run(trace);
  E e2(cfg, CostModel{}, opts);
  RunReport b = e2.run(trace);
  CHECK(a.to_json() == b.to_json());
  CHECK(a.csv_row() == b.csv_row());
  CHECK(a.gpu_hit_ratio >= 0.0);
  CHECK(a.gpu_hit_ratio <= a.total_hit_ratio);
  CHECK(a.total_hit_ratio <= 1.0);
  double step_sum = 0;
  for (double s : a.step_ms) step_sum += s;
  CHECK(approx(a.avg_latency_ms, step_sum, 1e-9));
  CHECK(approx(a.total_latency_ms, a.avg_latency_ms * double(a.batches), 1e-9));
  return fingerprint(e1, a);
}

// test_sim.cpp:170. The reference requires |dlogit| <= 1e-5 across modes in
// fp64; the B200 computes in bf16 / fp32, so its bars are relative to each
// request's logit scale: every mode within VALUE_REF_REL of the reference
// logits, and the B200 modes within VALUE_MODE_REL of each other.
constexpr double VALUE_REF_REL = 0.08, VALUE_MODE_REL = 0.02;

template <class E>
std::vector<std::vector<double>> value_run(Mode m, std::uint32_t batch, const std::vector<Request>& trace,
                                           const KVConfig& cfg, const ModelParams& params) {
  EngineOptions opts;
  opts.mode = m;
  opts.batch_size = batch;
  opts.model = &params;
  std::vector<std::vector<double>> logits;
  opts.logit_sink = &logits;
  E eng(cfg, CostModel{}, opts);
  eng.run(trace);
  return logits;
}

void sim_value_mode_invariant() {
  GenConfig g;
  g.num_users = 10;
  g.total_requests = 120;
  g.mean_final_len = 250;
  g.min_len = 10;
  g.max_len = 400;
  g.vocab = 32;
  g.candidates = 3;
  g.seed = 77;
  auto trace = generate_trace(g);
  KVConfig cfg;
  cfg.num_layers = 2;
  cfg.num_heads = 2;
  cfg.head_dim = 8;
  cfg.page_size = 16;
  cfg.chunk_size = 32;
  cfg.device_pages = 80;
  cfg.offload_quota = 128;
  ModelConfig mc;
  mc.num_layers = 2;
  mc.num_heads = 2;
  mc.head_dim = 8;
  mc.vocab = 32;
  mc.seed = 4;
  ModelParams params = ModelParams::random(mc);
  using RefV = mtkv::Engine<ValueBackend>;
  using B2V = mtkv::b200::Engine<ValueBackend>;
  const auto ref = value_run<RefV>(Mode::Hierarchical, 1, trace, cfg, params);
  std::vector<std::vector<std::vector<double>>> runs = {
      value_run<B2V>(Mode::Recompute, 1, trace, cfg, params), value_run<B2V>(Mode::GpuOnly, 1, trace, cfg, params),
      value_run<B2V>(Mode::Hierarchical, 1, trace, cfg, params),
      value_run<B2V>(Mode::Hierarchical, 3, trace, cfg, params)};
  double worst_ref = 0, worst_mode = 0;
  REQUIRE(ref.size() == trace.size());
  for (const auto& r : runs) REQUIRE(r.size() == trace.size());
  for (std::size_t i = 0; i < trace.size(); ++i) {
    double scale = 0;
    for (double x : ref[i]) scale = std::max(scale, std::fabs(x));
    for (const auto& r : runs)
      for (std::size_t j = 0; j < ref[i].size(); ++j) {
        worst_ref = std::max(worst_ref, std::fabs(r[i][j] - ref[i][j]) / scale);
        worst_mode = std::max(worst_mode, std::fabs(r[i][j] - runs[0][i][j]) / scale);
      }
  }
  std::printf("  value backend: worst |B200 - reference| %.3e, worst |mode - recompute| %.3e (of logit scale)\n",
              worst_ref, worst_mode);
  CHECK(worst_ref <= VALUE_REF_REL);
  CHECK(worst_mode <= VALUE_MODE_REL);
}

// -------------------------------------------------------- test_manager.cpp ---
KVConfig small_cfg(std::uint32_t pages) {
  KVConfig cfg;
  cfg.num_layers = 2;
  cfg.page_size = 8;
  cfg.chunk_size = 16;
  cfg.device_pages = pages;
  cfg.offload_quota = 64;
  return cfg;
}

Request req(UserId u, std::uint32_t delta, std::uint32_t cands = 1) {
  Request r;
  r.user = u;
  r.new_token_count = delta;
  r.candidate_count = cands;
  return r;
}

struct RefMgr {
  DevicePagedStore<TagBackend> dev;
  mtkv::CacheManager mgr;
  explicit RefMgr(const KVConfig& c) : dev(c.num_layers, c.device_pages, c.page_size), mgr(c, dev) {}
};
struct B2Mgr {
  mtkv::b200::CacheManager mgr;
  explicit B2Mgr(const KVConfig& c) : mgr(c) {}
};

std::string plans_str(const BatchMetadata& md) {
  std::string s;
  for (const auto& p : md.plans) {
    s += std::to_string(p.user) + ":" + std::to_string(p.history_len) + "," + std::to_string(p.reusable_len) + "," +
         std::to_string(p.device_served) + "," + std::to_string(p.host_onload) + "," +
         std::to_string(p.fresh_history) + "," + std::to_string(p.onload_chunks.size()) + "[";
    for (PageId x : p.scratch_pages) s += std::to_string(x) + " ";
    s += "];";
  }
  for (const auto& e : md.evictions)
    s += "ev" + std::to_string(e.user) + "," + std::to_string(e.freed_pages) + "," + std::to_string(e.tail_tokens_lost);
  return s;
}

template <class M>
std::string pages_str(M& mgr, UserId u) {
  std::string s = std::to_string(u) + ":";
  for (PageId p : mgr.user_pages(u)) s += std::to_string(p) + " ";
  return s;
}

template <class H>
std::string mgr_first_visit() {
  H h(small_cfg(64));
  auto& mgr = h.mgr;
  auto md = mgr.prepare_metadata({req(7, 20, 3)}, true);
  REQUIRE(md.plans.size() == 1);
  const auto& p = md.plans[0];
  CHECK(p.history_len == 0);
  CHECK(p.reusable_len == 0);
  CHECK(p.fresh_history == 0);
  CHECK(p.delta == 20);
  CHECK(p.fresh_tokens() == 23);
  CHECK(p.total_seq_len() == 23);
  CHECK(mgr.user_pages(7).size() == 3);
  CHECK(p.scratch_pages.size() == 1);
  CHECK(mgr.occupied_pages() == 4);
  mgr.finish_append(7, 20);
  CHECK(mgr.get_total_cache_length(7) == 20);
  CHECK(mgr.last_page_len(7) == 4);
  RequestPlan plan = md.plans[0];
  std::string fp = plans_str(md) + pages_str(mgr, 7);
  mgr.release_scratch(plan);
  CHECK(plan.scratch_pages.empty());
  CHECK(mgr.occupied_pages() == 3);
  return fp;
}

template <class H>
std::string mgr_resident() {
  H h(small_cfg(64));
  auto& mgr = h.mgr;
  auto md1 = mgr.prepare_metadata({req(1, 16)}, true);
  mgr.finish_append(1, 16);
  mgr.release_scratch(md1.plans[0]);
  auto md2 = mgr.prepare_metadata({req(1, 10)}, true);
  const auto& p = md2.plans[0];
  CHECK(p.history_len == 16);
  CHECK(p.device_served == 16);
  CHECK(p.host_onload == 0);
  CHECK(p.fresh_history == 0);
  CHECK(p.fresh_tokens() == 11);
  return plans_str(md1) + plans_str(md2) + pages_str(mgr, 1);
}

template <class H>
std::string mgr_same_user_twice() {
  H h(small_cfg(64));
  auto& mgr = h.mgr;
  auto md = mgr.prepare_metadata({req(4, 10), req(4, 6)}, true);
  CHECK(md.plans[0].history_len == 0);
  CHECK(md.plans[1].history_len == 10);
  CHECK(md.plans[1].device_served == 10);
  CHECK(md.plans[1].fresh_history == 0);
  return plans_str(md) + pages_str(mgr, 4);
}

template <class H>
std::string mgr_round_robin() {
  H h(small_cfg(5));
  auto& mgr = h.mgr;
  std::string fp;
  for (UserId u : {1, 2}) {
    auto md = mgr.prepare_metadata({req(u, 16)}, true);
    mgr.finish_append(u, 16);
    mgr.release_scratch(md.plans[0]);
    fp += plans_str(md);
  }
  CHECK(mgr.occupied_pages() == 4);
  auto md = mgr.prepare_metadata({req(3, 16)}, true);
  REQUIRE(md.evictions.size() >= 1);
  CHECK(md.evictions[0].user == 1);
  CHECK(md.evictions[0].tail_tokens_lost == 16);
  CHECK(mgr.find(1)->device_len == 0);
  CHECK(mgr.user_pages(1).empty());
  CHECK(mgr.counters().evictions == 1);
  mgr.finish_append(3, 16);
  mgr.release_scratch(md.plans[0]);
  return fp + plans_str(md) + pages_str(mgr, 3);
}

template <class H>
std::string mgr_zero_copy() {
  const KVConfig cfg = small_cfg(64);
  H h(cfg);
  auto& mgr = h.mgr;
  auto md = mgr.prepare_metadata({req(5, 40)}, true);
  mgr.finish_append(5, 40);
  mgr.release_scratch(md.plans[0]);
  mgr.advance_persisted(5, 32);
  auto freed = mgr.evict_user(5);
  CHECK(freed.size() == 5);
  CHECK(mgr.counters().tail_tokens_lost == 8);
  CHECK(mgr.find(5)->persisted_len == 32);
  CHECK(mgr.find(5)->device_len == 0);
  CHECK(mgr.get_total_cache_length(5) == 32);
  auto md2 = mgr.prepare_metadata({req(5, 10)}, true);
  const auto& p = md2.plans[0];
  CHECK(p.history_len == 40);
  CHECK(p.host_onload == 32);
  CHECK(p.onload_chunks == std::vector<std::uint64_t>{0, 1});
  CHECK(p.fresh_history == 8);
  mgr.commit_onload(5, p);
  CHECK(mgr.find(5)->device_len == 32);
  std::string fp = plans_str(md) + plans_str(md2) + pages_str(mgr, 5);
  for (PageId x : freed) fp += std::to_string(x) + ",";
  // without the host tier the whole history is fresh
  H h2(cfg);
  auto& mgr2 = h2.mgr;
  auto mda = mgr2.prepare_metadata({req(6, 40)}, false);
  mgr2.finish_append(6, 40);
  mgr2.release_scratch(mda.plans[0]);
  mgr2.evict_user(6);
  auto mdb = mgr2.prepare_metadata({req(6, 10)}, false);
  CHECK(mdb.plans[0].fresh_history == 40);
  CHECK(mdb.plans[0].host_onload == 0);
  return fp + plans_str(mda) + plans_str(mdb);
}

template <class H>
std::string mgr_locking() {
  H h(small_cfg(8));
  auto& mgr = h.mgr;
  auto md = mgr.prepare_metadata({req(1, 16)}, true);
  mgr.finish_append(1, 16);
  mgr.release_scratch(md.plans[0]);
  mgr.lock_user(1);
  CHECK(mgr.is_locked(1));
  CHECK_THROWS_AS(mgr.lock_user(1), Error);
  CHECK_THROWS_AS(mgr.evict_user(1), Error);
  CHECK_THROWS_AS(mgr.lock_user(42), Error);
  CHECK_THROWS_AS(mgr.prepare_metadata({req(2, 48)}, true), BatchRejected);
  mgr.unlock_user(1);
  CHECK_FALSE(mgr.is_locked(1));
  CHECK_THROWS_AS(mgr.unlock_user(1), Error);
  auto md2 = mgr.prepare_metadata({req(2, 56)}, true);
  CHECK(md2.evictions.size() == 1);
  CHECK(md2.evictions[0].user == 1);
  return plans_str(md) + plans_str(md2) + pages_str(mgr, 2);
}

template <class H>
std::string mgr_oversized() {
  H h(small_cfg(4));
  CHECK_THROWS_AS(h.mgr.prepare_metadata({req(1, 100)}, true), BatchRejected);
  return "";
}

template <class H>
std::string mgr_batch_protects() {
  H h(small_cfg(6));
  auto& mgr = h.mgr;
  std::string fp;
  for (UserId u : {1, 2}) {
    auto md = mgr.prepare_metadata({req(u, 16)}, true);
    mgr.finish_append(u, 16);
    mgr.release_scratch(md.plans[0]);
    fp += plans_str(md);
  }
  CHECK_THROWS_AS(mgr.prepare_metadata({req(1, 8), req(2, 8)}, true), BatchRejected);
  return fp;
}

// runs a case for both implementations and compares what they observed
void both(const char* name, const std::function<std::string()>& ref, const std::function<std::string()>& b200) {
  g_case = std::string(name) + " (reference)";
  const int f0 = g_failed;
  std::string a, b;
  try {
    a = ref();
  } catch (const std::exception& e) {
    ++g_failed;
    std::printf("FAIL [%s] threw: %s\n", g_case.c_str(), e.what());
  }
  g_case = std::string(name) + " (b200)";
  try {
    b = b200();
  } catch (const std::exception& e) {
    ++g_failed;
    std::printf("FAIL [%s] threw: %s\n", g_case.c_str(), e.what());
  }
  g_case = name;
  ++g_checks;
  if (a != b) {
    ++g_failed;
    std::printf("FAIL [%s] observable results differ:\n  reference: %.300s\n  b200:      %.300s\n", name, a.c_str(),
                b.c_str());
  }
  std::printf("%s %s\n", g_failed == f0 ? "ok  " : "FAIL", name);
}

}  // namespace

int main(int argc, char** argv) {
  const bool engine = argc > 1 && std::strcmp(argv[1], "--engine") == 0;
  both("manager: first visit plans fresh-only with scratch", mgr_first_visit<RefMgr>, mgr_first_visit<B2Mgr>);
  both("manager: resident prefix served from the device tier", mgr_resident<RefMgr>, mgr_resident<B2Mgr>);
  both("manager: same user twice plans against projected state", mgr_same_user_twice<RefMgr>,
       mgr_same_user_twice<B2Mgr>);
  both("manager: round-robin over capacity evicts the least recent", mgr_round_robin<RefMgr>, mgr_round_robin<B2Mgr>);
  both("manager: zero-copy eviction keeps the persisted prefix", mgr_zero_copy<RefMgr>, mgr_zero_copy<B2Mgr>);
  both("manager: locking protocol", mgr_locking<RefMgr>, mgr_locking<B2Mgr>);
  both("manager: oversized batches are rejected up front", mgr_oversized<RefMgr>, mgr_oversized<B2Mgr>);
  both("manager: batch members protect each other", mgr_batch_protects<RefMgr>, mgr_batch_protects<B2Mgr>);
  if (engine) {
    both("sim: empty trace yields a zeroed report", sim_empty<RefTag>, sim_empty<B2Tag>);
    both("sim: resident prefix second visit is a full device hit", sim_resident<RefTag>, sim_resident<B2Tag>);
    both("sim: unlimited capacity chunk=page total hit 100%", sim_unlimited<RefTag>, sim_unlimited<B2Tag>);
    both("sim: two-user alternating eviction (hierarchical)", [] { return sim_alternating<RefTag>(Mode::Hierarchical); },
         [] { return sim_alternating<B2Tag>(Mode::Hierarchical); });
    both("sim: two-user alternating eviction (gpu_only)", [] { return sim_alternating<RefTag>(Mode::GpuOnly); },
         [] { return sim_alternating<B2Tag>(Mode::GpuOnly); });
    both("sim: tokens processed across modes", sim_tokens_across_modes<RefTag>, sim_tokens_across_modes<B2Tag>);
    both("sim: gpu hit ratios agree between gpu_only and hierarchical", sim_hit_ratios_agree<RefTag>,
         sim_hit_ratios_agree<B2Tag>);
    both("sim: report invariants and determinism", sim_determinism<RefTag>, sim_determinism<B2Tag>);
    g_case = "sim: value backend logits are mode-invariant";
    const int f0 = g_failed;
    try {
      sim_value_mode_invariant();
    } catch (const std::exception& e) {
      ++g_failed;
      std::printf("FAIL [%s] threw: %s\n", g_case.c_str(), e.what());
    }
    std::printf("%s %s\n", g_failed == f0 ? "ok  " : "FAIL", g_case.c_str());
  }
  std::printf("%d checks, %d failed\n", g_checks, g_failed);
  return g_failed ? 1 : 0;
}
