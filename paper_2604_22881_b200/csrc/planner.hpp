// Host control plane of the B200 serving path.
//
// The reference splits decisions across CacheManager (manager.cpp), Pipeline
// (pipeline.cpp) and Engine<B> (sim.hpp). Here they form one deterministic
// planner that turns a batch of requests into a BatchWork list — the exact
// set of copies, scatters, appends, attention spans and offloads the GPU
// executor must run — without ever waiting for the device. Every decision
// (hit class, eviction order, page ids, lock/quota/persistence timing on the
// simulated clock) is bit-identical to the reference; tests/test_planner.py
// replays traces against the reference and the C oracle.
//
// Data layout is flat and index-based so the same tables can be mirrored to
// the device: users live in a dense slot array (id -> slot hash), recency is
// an intrusive doubly-linked list over slots, free device pages are a LIFO
// id stack (reference free-list order, store.hpp:63).
#pragma once

#include <cstdint>
#include <queue>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/mtkv_b200.h"
#include "devctl.hpp"

namespace mtkv_b200 {

struct Error {
  int code;
  std::string msg;
};

struct UserRec {
  uint32_t id = 0;
  bool known = false;      // has a sequence-table entry (manager.cpp:200 state())
  bool has_pages = false;  // has a page-table entry
  bool locked = false;
  bool in_lru = false;
  uint64_t total_len = 0, device_len = 0, persisted_len = 0, last_access = 0;
  uint64_t recompute_len = 0;
  uint32_t pending = 0;
  int32_t newer = -1, older = -1;     // recency links
  std::vector<uint32_t> pages;        // logical page -> physical page id
  std::vector<uint64_t> host_chunks;  // persisted chunk ids, in chunk order
  std::vector<uint32_t> tokens;       // full token history (value backend)
};

// One request's share of a batch, in executor terms.
struct ReqWork {
  uint32_t slot = 0;
  mtkv_request_plan plan{};
  uint64_t start = 0;          // first fresh position (device_len when encoding)
  uint32_t n_hist = 0;         // fresh history rows appended (lost tail + delta)
  uint32_t pages_off = 0, n_pages = 0;      // into BatchWork::pages (user page snapshot)
  uint32_t scratch_off = 0, n_scratch = 0;  // into BatchWork::pages
  uint32_t tok_off = 0;        // into BatchWork::tokens: fresh history ids ++ candidate ids
  bool recompute_prefix = false;  // adaptive onload policy: host-hit prefix re-encoded (start = 0)
  // adaptive policy, split host hit: the prefix's first head_chunks chunks are
  // re-encoded (positions [0, head_rows), their ids at head_tok_off in
  // BatchWork::tokens: the executor runs them as an extra request ahead of this
  // one's attention), the remaining chunks are onloaded
  uint32_t head_chunks = 0, head_rows = 0, head_tok_off = 0;
};

struct ChunkMove {
  uint64_t chunk_id = 0;   // host-store chunk id (executor maps to pinned memory)
  uint32_t user = 0;
  uint32_t chunk_index = 0;
  uint32_t pages_off = 0;  // pages_per_chunk ids in BatchWork::pages
};

struct BatchWork {
  int rc = MTKV_OK;
  std::string error;
  std::vector<ReqWork> reqs;
  std::vector<uint32_t> pages;
  std::vector<uint32_t> tokens;
  std::vector<ChunkMove> onloads;     // host -> device, in reference staging order
  std::vector<ChunkMove> offloads;    // device -> host, triggered after compute
  std::vector<uint64_t> persisted;    // chunk ids whose completion fired at batch start
  std::vector<mtkv_eviction> evictions;
  uint64_t fresh_rows = 0;            // sum of fresh history + candidates
  double sim_start = 0, sim_end = 0;
};

class Planner {
 public:
  Planner(const mtkv_kv_config& kv, const mtkv_cost_model& cost, int mode, bool keep_tokens);

  // One batch: process_due, prepare_metadata, schedule, commit, append
  // bookkeeping, scratch release, offload triggers (sim.hpp:332).
  void plan_batch(const mtkv_request* reqs, uint32_t n, BatchWork& out);
  void drain(std::vector<uint64_t>* persisted = nullptr);

  // manager surface
  int evict(uint32_t user, std::string& err);
  // CacheManager step surface (manager.hpp:103-126); request indices refer to
  // the last mgr_prepare
  int mgr_prepare(const mtkv_request* reqs, uint32_t n, bool host_enabled, std::string& err);
  const std::vector<uint32_t>* mgr_scratch(uint32_t i) const;
  int mgr_release_pages(const uint32_t* pages, uint32_t n, std::string& err);
  int mgr_commit_onload(uint32_t user, uint64_t reusable_len, uint32_t onload_chunks, std::string& err);
  int mgr_finish_append(uint32_t user, uint64_t appended, std::string& err);
  int mgr_advance_persisted(uint32_t user, uint64_t tokens, std::string& err);
  int mgr_lock(uint32_t user, bool lock, std::string& err);
  uint32_t last_page_len(uint32_t user) const;
  const UserRec* find(uint32_t user) const;
  std::vector<uint32_t> known_users() const;
  std::vector<uint32_t> lru_snapshot() const;
  void report(mtkv_run_report& r) const;
  const BatchWork& last() const { return last_; }
  void keep_last(const BatchWork& w) { last_ = w; }
  uint64_t chunk_bytes_exact() const { return chunk_bytes_u64_; }
  const mtkv_kv_config& kv() const { return kv_; }
  int mode() const { return mode_; }
  uint32_t pages_per_chunk() const { return kv_.chunk_size / kv_.page_size; }
  uint64_t chunks_created() const { return next_chunk_id_; }
  // Device control plane (devctl.hpp): prepare_metadata's decisions come from the
  // GPU; this planner mirrors them and sends its own state changes back.
  void set_device_ctl(DevCtl* c) { ctl_ = c; }
  // Executor policy for host hits (mtkv_engine_options::onload_policy): which
  // prefixes come back over the host link and which are re-encoded on the SMs.
  // Decisions of the control plane are unaffected.
  void set_onload_policy(int policy, double link_bytes_per_s, double recompute_tok_per_s) {
    policy_ = policy;
    link_Bps_ = link_bytes_per_s;
    recompute_tps_ = recompute_tok_per_s;
  }
  bool device_ctl() const { return ctl_ != nullptr; }

 private:
  int slot_of(uint32_t id, bool create);
  void lru_unlink(int s);
  void lru_front(int s);
  uint32_t pop_page();
  void push_page(uint32_t p);
  bool evict_slot(int s, uint64_t* freed, std::string& err);
  int free_pages_for(uint64_t need, const std::vector<char>& in_batch, BatchWork& w);
  bool prepare_metadata(const mtkv_request* reqs, uint32_t n, bool hier, std::vector<int>& slot,
                        std::vector<uint32_t>& scratch_ids, BatchWork& w);
  bool prepare_on_device(const mtkv_request* reqs, uint32_t n, std::vector<int>& slot,
                         std::vector<uint32_t>& scratch_ids, BatchWork& w);
  void note_update(int s);  // persisted length / lock bit changed on the host
  void fire_completions(double now, std::vector<uint64_t>* persisted, BatchWork* w);
  void schedule_onload(double submit, size_t n_chunks, std::vector<double>& fire);
  double schedule_offload(double submit);
  void trigger_offloads(int s, double t, BatchWork& w);

  mtkv_kv_config kv_;
  mtkv_cost_model cost_;
  int mode_;
  bool keep_tokens_;
  std::vector<UserRec> users_;
  std::unordered_map<uint32_t, int> index_;
  int newest_ = -1, oldest_ = -1;
  std::vector<uint32_t> free_;      // back = next page handed out
  uint64_t occupied_ = 0, stamp_ = 0, evictions_ = 0, tail_lost_ = 0, pages_allocated_ = 0;
  uint64_t host_total_ = 0;
  uint64_t next_chunk_id_ = 0;

  // event schedule (pipeline.cpp) on simulated seconds
  double chunk_bytes_ = 0;
  uint64_t chunk_bytes_u64_ = 0;
  double host_cpu_free_ = 0, h2d_free_ = 0, scatter_free_ = 0, offload_free_ = 0;
  double pinned_free_[2] = {0, 0};
  uint64_t pinned_turn_ = 0;
  struct Pending {
    double done;
    uint64_t order;
    int slot;
    uint64_t chunk_index, chunk_id;
  };
  struct Later {
    bool operator()(const Pending& a, const Pending& b) const {
      return a.done > b.done || (a.done == b.done && a.order > b.order);
    }
  };
  std::priority_queue<Pending, std::vector<Pending>, Later> pending_;
  uint64_t order_ = 0;
  uint64_t quota_used_ = 0;

  // report accumulators (sim.hpp:203-208)
  double clock_ = 0, steps_[9] = {0}, wait_ = 0, comp_ = 0, latency_ = 0;
  uint64_t required_ = 0, dev_served_ = 0, host_served_ = 0, processed_ = 0, requests_ = 0,
           batches_ = 0, peak_pages_ = 0;
  BatchWork last_;
  std::vector<std::vector<uint32_t>> mgr_scratch_;  // step surface: scratch ids per request
  DevCtl* ctl_ = nullptr;
  int policy_ = MTKV_ONLOAD_ALWAYS;
  double link_Bps_ = 54e9, recompute_tps_ = 38e6;
  uint64_t prefix_onloaded_ = 0, prefix_recomputed_ = 0;
  void choose_recompute(BatchWork& w);
  std::vector<CtlUpd> ctl_upd_;  // host-side changes queued for the next device prepare
  std::unordered_map<int, size_t> ctl_upd_at_;
};

}  // namespace mtkv_b200
