// Device-side control plane: the batched user lookup, LRU-recency update,
// eviction-victim selection and LIFO page allocation of the reference's
// CacheManager::prepare_metadata (manager.cpp:74-139, ensure_free :55,
// evict_user :141), plus the end-of-batch commit_onload / finish_append /
// release_scratch (:178-202), executed by one CTA on the B200 over
// device-resident tables.
//
// Tables (HBM): an open-addressing user-id -> slot hash; per slot the lengths,
// the recency stamp, lock / LRU flags and a fixed-capacity page list; the free
// page stack. The LRU list of the reference is the order of recency stamps of
// the users that are "in the list" (a touch moves a user to the front with a
// fresh, strictly larger stamp; an eviction removes it), so victim selection is
// "smallest stamps first" among in-list, unlocked users not in the batch: a
// weighted radix select finds the stamp threshold at which the freed pages
// cover the batch's deficit, warp ballots compact the victims, a bitonic sort
// orders them, and one warp replays the interleaved evict-push / allocate-pop
// sequence so page ids come out exactly as the reference's free list hands
// them out.
//
// The host planner keeps a mirror it updates from the kernel's output (page
// lists, victims, stamps) and owns the simulated-clock schedule; persisted
// lengths and lock bits it changes between batches are sent as updates.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace mtkv_b200 {

struct CtlReq {
  uint32_t user, delta, ncand, pad;
};
struct CtlUpd {  // host-side change since the last batch
  uint32_t slot, locked;
  uint64_t persisted_len;
};
struct CtlPlan {  // per request
  int32_t slot;
  uint32_t onload_chunks;
  uint32_t grow_off, grow_n;        // into CtlHdr-following id array
  uint32_t scratch_off, scratch_n;
  uint64_t stamp;
  uint64_t history_len, device_served, host_onload, reusable_len, fresh_history;
};
struct CtlEvict {
  uint32_t slot, user, freed_pages, pad;
  uint64_t tail_lost;
};
enum CtlFail : int32_t { CTL_OK = 0, CTL_REJECT_PAGES = 1, CTL_REJECT_VICTIMS = 2, CTL_BAD_REQUEST = 3, CTL_CAPACITY = 4, CTL_STAGING = 5 };
struct CtlHdr {
  int32_t fail;      // CtlFail
  int32_t fail_at;   // request index of the failure (touched, not allocated)
  uint32_t n_evict, n_ids, free_top, n_slots;
  uint64_t stamp;
};

class DevCtl {
 public:
  // page_size/chunk_size/device_pages: KVConfig; hier: host tier enabled
  int init(uint32_t device_pages, uint32_t page_size, uint32_t chunk_size, bool hier, uint32_t max_users,
           uint32_t max_pages_per_user, uint64_t staging_tokens, std::string& err);
  ~DevCtl();
  // One batch: updates, then prepare + commit + append + scratch release on the
  // device; blocks until the decisions are back on the host.
  int prepare(const CtlReq* reqs, uint32_t n, const std::vector<CtlUpd>& upd, std::string& err);
  const CtlHdr& hdr() const { return hdr_; }
  const CtlPlan* plans() const { return plans_; }
  const CtlEvict* evictions() const { return evict_; }
  const uint32_t* ids() const { return ids_; }
  double last_kernel_ms() const { return last_ms_; }
  uint32_t max_users() const { return max_users_; }

 private:
  uint32_t device_pages_ = 0, page_size_ = 0, chunk_size_ = 0, max_users_ = 0, max_pages_ = 0, hash_cap_ = 0;
  bool hier_ = false;
  uint64_t staging_tokens_ = 0;
  cudaStream_t st_ = nullptr;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  void* state_ = nullptr;  // device tables
  size_t state_bytes_ = 0;
  void* io_dev_ = nullptr;  // per-batch inputs + outputs (device)
  char* io_host_ = nullptr; // pinned mirror
  size_t io_bytes_ = 0;
  CtlHdr hdr_{};
  CtlPlan* plans_ = nullptr;
  CtlEvict* evict_ = nullptr;
  uint32_t* ids_ = nullptr;
  double last_ms_ = 0;
};

}  // namespace mtkv_b200
