// Drop-in C++ front end of the B200 serving path for code written against the
// reference library (`mtkv::`, /root/reference/proj/core/include/mtkv).
//
//   #include <mtkv/sim.hpp>              // the reference's types
//   #include "mtkv_b200_engine.hpp"
//   mtkv::b200::Engine<mtkv::TagBackend> eng(cfg, cost, opts);   // was mtkv::Engine<TagBackend>
//
// Every class takes and returns the reference's own types (KVConfig,
// CostModel, EngineOptions, Request, RunReport, RequestPlan, BatchMetadata,
// SequenceState, ...) and throws the reference's exceptions (mtkv::Error,
// mtkv::BatchRejected) with the reference's messages. Underneath is the C-ABI
// of include/mtkv_b200.h (libmtkv_b200.so): the control plane runs on the host
// planner, payloads live in the B200's paged HBM pool / pinned host tier.
//
//   mtkv::b200::Engine<B>      <- mtkv::Engine<B>      (sim.hpp:110)
//   mtkv::b200::CacheManager   <- mtkv::CacheManager   (manager.hpp:89)
//
// Differences a caller can observe:
//   * Engine<ValueBackend> regenerates the model weights on the device from
//     opts.model->cfg (the reference init, model.cpp:34, same RNG streams);
//     arbitrary hand-set ModelParams are not uploaded. Logits are fp32 from
//     bf16 tensor-core math (tolerance: DESIGN.md (c)).
//   * device() / host() / quota() are read-only views (free_count, chunk_count,
//     in_flight): the stores themselves are GPU / pinned memory.
//   * CacheManager owns its page free list (the reference's takes a
//     PageAllocator&): same LIFO order, page 0 handed out first.
//   * event_sink (TraceEvent) is not produced.
#pragma once

#include <map>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include <mtkv/sim.hpp>

#include "mtkv_b200.h"

namespace mtkv {
namespace b200 {

namespace detail {

inline mtkv_kv_config to_c(const KVConfig& c) {
  return mtkv_kv_config{c.num_layers,  c.num_heads,         c.head_dim,      c.page_size,    c.chunk_size,
                        c.device_pages, c.onload_pages,     c.bytes_per_element, c.offload_quota, c.host_capacity};
}

inline mtkv_cost_model to_c(const CostModel& k) {
  return mtkv_cost_model{k.bus_bandwidth, k.tx_setup,     k.host_bandwidth, k.page_op,      k.attn_coeff,
                         k.linear_coeff,  k.embed_coeff,  k.layout_coeff,   k.meta_fixed,   k.strip_fixed,
                         k.embed_fixed,   k.layout_fixed, k.await_fixed,    k.update_fixed, k.commit_per_chunk,
                         k.offload_submit, k.post_fixed};
}

inline void check(int rc) {
  if (rc == MTKV_OK) return;
  const std::string msg = mtkv_last_error();
  if (rc == MTKV_BATCH_REJECTED) throw BatchRejected(msg);
  throw Error(msg);
}

// Request vectors -> C structs; the id arrays stay owned by `batch`
inline std::vector<mtkv_request> to_c(const std::vector<Request>& batch) {
  std::vector<mtkv_request> r(batch.size());
  for (size_t i = 0; i < batch.size(); ++i) {
    const Request& q = batch[i];
    r[i].timestamp = q.timestamp;
    r[i].user = q.user;
    r[i].new_token_count = q.delta();
    r[i].candidate_count = q.num_candidates();
    r[i].new_tokens = q.new_tokens.empty() ? nullptr : q.new_tokens.data();
    r[i].candidates = q.candidates.empty() ? nullptr : q.candidates.data();
  }
  return r;
}

// read-only manager surface shared by Engine::manager() and CacheManager
class ManagerView {
 public:
  ManagerView(const void* obj, int is_engine) : obj_(obj), eng_(is_engine) {}

  std::vector<UserId> known_users() const {
    std::vector<UserId> out(mtkv_known_users(obj_, eng_, nullptr, 0));
    mtkv_known_users(obj_, eng_, out.data(), uint32_t(out.size()));
    return out;
  }
  // manager.cpp:40; the pointer stays valid until the next call for the same user
  const SequenceState* find(UserId user) const {
    mtkv_sequence_state s;
    if (mtkv_user_state(obj_, eng_, user, &s) != MTKV_OK) return nullptr;
    SequenceState& out = seq_[user];
    out.total_len = s.total_len;
    out.device_len = s.device_len;
    out.persisted_len = s.persisted_len;
    out.locked = s.locked != 0;
    out.last_access = s.last_access;
    return &out;
  }
  const std::vector<PageId>& user_pages(UserId user) const {  // manager.cpp:203
    std::vector<PageId>& v = pages_[user];
    v.assign(mtkv_user_pages(obj_, eng_, user, nullptr, 0), 0);
    mtkv_user_pages(obj_, eng_, user, v.data(), uint32_t(v.size()));
    return v;
  }
  bool is_locked(UserId user) const { return mtkv_is_locked(obj_, eng_, user) != 0; }
  std::uint64_t get_total_cache_length(UserId user) const { return mtkv_get_total_cache_length(obj_, eng_, user); }
  std::uint64_t occupied_pages() const { return report().occupied_pages; }
  ManagerCounters counters() const {
    const mtkv_run_report r = report();
    ManagerCounters c;
    c.evictions = r.evictions;
    c.tail_tokens_lost = r.tail_tokens_lost;
    c.pages_allocated = r.pages_allocated;
    return c;
  }
  struct Lru {  // manager.hpp:25 LruIndex, read side
    std::vector<UserId> order;
    std::vector<UserId> snapshot() const { return order; }
    bool contains(UserId u) const {
      for (UserId x : order)
        if (x == u) return true;
      return false;
    }
    std::size_t size() const { return order.size(); }
  };
  Lru lru() const {
    Lru l;
    l.order.resize(mtkv_lru_snapshot(obj_, eng_, nullptr, 0));
    mtkv_lru_snapshot(obj_, eng_, l.order.data(), uint32_t(l.order.size()));
    return l;
  }
  std::vector<PageId> evict_user(UserId user) {  // manager.cpp:141, returns the freed pages
    std::vector<PageId> freed = user_pages(user);
    check(mtkv_evict_user(const_cast<void*>(obj_), eng_, user));
    return freed;
  }

 protected:
  mtkv_run_report report() const {
    mtkv_run_report r;
    check(mtkv_report(obj_, eng_, &r));
    return r;
  }
  const void* obj_;
  int eng_;
  mutable std::map<UserId, SequenceState> seq_;
  mutable std::map<UserId, std::vector<PageId>> pages_;
};

}  // namespace detail

/// manager.hpp:89 CacheManager on the B200 path's host control plane (the
/// same object the engine runs ahead of the GPU).
class CacheManager : public detail::ManagerView {
 public:
  explicit CacheManager(const KVConfig& cfg) : detail::ManagerView(nullptr, 0), cfg_(cfg) {
    const mtkv_kv_config kv = detail::to_c(cfg);
    const mtkv_cost_model cm = detail::to_c(CostModel{});
    p_ = mtkv_planner_create(&kv, &cm, MTKV_MODE_HIERARCHICAL);
    if (!p_) throw Error(mtkv_last_error());
    obj_ = p_;
  }
  ~CacheManager() { mtkv_planner_destroy(p_); }
  CacheManager(const CacheManager&) = delete;
  CacheManager& operator=(const CacheManager&) = delete;

  const KVConfig& config() const { return cfg_; }

  BatchMetadata prepare_metadata(const std::vector<Request>& batch, bool host_enabled) {  // manager.cpp:74
    std::vector<mtkv_request> r = detail::to_c(batch);
    const int rc = mtkv_planner_prepare_metadata(p_, r.data(), uint32_t(r.size()), host_enabled ? 1 : 0);
    detail::check(rc);
    BatchMetadata md;
    std::vector<mtkv_request_plan> pl(mtkv_last_plans(p_, 0, nullptr, 0));
    mtkv_last_plans(p_, 0, pl.data(), uint32_t(pl.size()));
    for (uint32_t i = 0; i < pl.size(); ++i) {
      RequestPlan p;
      p.user = pl[i].user;
      p.history_len = pl[i].history_len;
      p.reusable_len = pl[i].reusable_len;
      p.device_served = pl[i].device_served;
      p.host_onload = pl[i].host_onload;
      p.fresh_history = pl[i].fresh_history;
      p.delta = pl[i].delta;
      p.num_candidates = pl[i].num_candidates;
      for (uint64_t c = 0; c < pl[i].onload_chunks; ++c) p.onload_chunks.push_back(c);
      p.scratch_pages.resize(mtkv_planner_scratch_pages(p_, i, nullptr, 0));
      mtkv_planner_scratch_pages(p_, i, p.scratch_pages.data(), uint32_t(p.scratch_pages.size()));
      md.plans.push_back(std::move(p));
    }
    std::vector<mtkv_eviction> ev(mtkv_last_evictions(p_, 0, nullptr, 0));
    mtkv_last_evictions(p_, 0, ev.data(), uint32_t(ev.size()));
    for (const mtkv_eviction& e : ev) md.evictions.push_back(EvictionRecord{e.user, e.freed_pages, e.tail_tokens_lost});
    return md;
  }
  void lock_user(UserId user) { detail::check(mtkv_planner_lock_user(p_, user)); }
  void unlock_user(UserId user) { detail::check(mtkv_planner_unlock_user(p_, user)); }
  void commit_onload(UserId user, const RequestPlan& plan) {
    detail::check(mtkv_planner_commit_onload(p_, user, plan.reusable_len, uint32_t(plan.onload_chunks.size())));
  }
  void finish_append(UserId user, std::uint64_t appended) {
    detail::check(mtkv_planner_finish_append(p_, user, appended));
  }
  void advance_persisted(UserId user, std::uint64_t tokens) {
    detail::check(mtkv_planner_advance_persisted(p_, user, tokens));
  }
  void release_scratch(RequestPlan& plan) {
    detail::check(mtkv_planner_release_scratch(p_, plan.scratch_pages.data(), uint32_t(plan.scratch_pages.size())));
    plan.scratch_pages.clear();
  }
  std::uint32_t last_page_len(UserId user) const { return mtkv_planner_last_page_len(p_, user); }

 private:
  KVConfig cfg_;
  mtkv_planner* p_ = nullptr;
};

/// sim.hpp:110 Engine<B> with the data plane on a B200.
template <class B>
class Engine {
  static constexpr bool kValue = std::is_same_v<B, ValueBackend>;

 public:
  Engine(const KVConfig& cfg, const CostModel& cost, const EngineOptions& opts) : opts_(opts), view_(nullptr, 1) {
    cfg.validate();
    cost.validate();
    mtkv_engine_options eo{};
    eo.mode = int(opts.mode);  // Mode enum order matches (sim.hpp:25)
    eo.backend = kValue ? MTKV_BACKEND_VALUE : MTKV_BACKEND_TAG;
    eo.batch_size = opts.batch_size;
    eo.seed = opts.seed;
    if constexpr (kValue) {
      MTKV_CHECK(opts.model != nullptr, "value backend requires model params");
      MTKV_CHECK(opts.model->cfg.num_layers == cfg.num_layers && opts.model->cfg.hidden() == cfg.hidden(),
                 "value backend: model dimensions disagree with cache config");
      const ModelConfig& m = opts.model->cfg;
      eo.model = mtkv_model_config{m.num_layers, m.num_heads, m.head_dim, m.vocab, m.seed};
      eo.keep_logits = opts.logit_sink ? 1 : 0;
      vocab_ = m.vocab;
    }
    const mtkv_kv_config kv = detail::to_c(cfg);
    const mtkv_cost_model cm = detail::to_c(cost);
    e_ = mtkv_engine_create(&kv, &cm, &eo);
    if (!e_) throw Error(mtkv_last_error());
    view_ = detail::ManagerView(e_, 1);
    cfg_pages_ = cfg.device_pages;
  }
  ~Engine() { mtkv_engine_destroy(e_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  RunReport run(const std::vector<Request>& trace) {  // sim.hpp:135
    for (const auto& batch : batchify(trace, opts_.batch_size)) process_batch(batch);
    drain();
    return report();
  }

  void process_batch(const std::vector<Request>& batch) {  // sim.hpp:332
    std::vector<mtkv_request> r = detail::to_c(batch);
    detail::check(mtkv_engine_process_batch(e_, r.data(), uint32_t(r.size())));
    if constexpr (kValue) {
      if (opts_.logit_sink && !batch.empty()) {  // logit_sink: one vector per request
        std::vector<float> l(batch.size() * vocab_);
        if (mtkv_engine_last_logits(e_, l.data(), uint32_t(batch.size())) < 0) throw Error(mtkv_last_error());
        for (size_t i = 0; i < batch.size(); ++i)
          opts_.logit_sink->emplace_back(l.begin() + i * vocab_, l.begin() + (i + 1) * vocab_);
      }
    }
  }

  void drain() { detail::check(mtkv_engine_drain(e_)); }  // sim.hpp:145

  RunReport report() const {  // sim.hpp:457
    mtkv_run_report x;
    detail::check(mtkv_report(e_, 1, &x));
    RunReport r;
    r.mode = mode_name(opts_.mode);
    r.backend = kValue ? "value" : "tag";
    r.batch_size = opts_.batch_size;
    r.seed = opts_.seed;
    for (size_t i = 0; i < r.step_ms.size(); ++i) r.step_ms[i] = x.step_ms[i];
    r.wait_ms = x.wait_ms;
    r.comp_ms = x.comp_ms;
    r.gpu_hit_ratio = x.gpu_hit_ratio;
    r.total_hit_ratio = x.total_hit_ratio;
    r.tokens_processed = x.tokens_processed;
    r.evictions = x.evictions;
    r.tail_tokens_lost = x.tail_tokens_lost;
    r.requests = x.requests;
    r.batches = x.batches;
    r.avg_latency_ms = x.avg_latency_ms;
    r.total_latency_ms = x.total_latency_ms;
    r.peak_pages = x.peak_pages;
    return r;
  }

  detail::ManagerView& manager() { return view_; }  // sim.hpp:149

  struct DeviceView {  // DevicePagedStore read side (store.hpp:54)
    const Engine* e;
    std::size_t free_count() const { return e->raw_report().free_pages; }
    std::uint32_t num_pages() const { return e->cfg_pages_; }
  };
  struct HostView {  // HostChunkedStore read side (store.hpp:150)
    const Engine* e;
    std::uint64_t chunk_count(UserId u) const {
      mtkv_sequence_state s;
      return mtkv_user_state(e->e_, 1, u, &s) == MTKV_OK ? s.host_chunks : 0;
    }
  };
  DeviceView device() const { return DeviceView{this}; }
  HostView host() const { return HostView{this}; }
  OffloadQuota quota() const {
    OffloadQuota q;
    q.in_flight = raw_report().quota_in_flight;
    return q;
  }
  double clock() const { return raw_report().clock; }
  std::uint64_t pending_offload_chunks(UserId u) const {
    mtkv_sequence_state s;
    return mtkv_user_state(e_, 1, u, &s) == MTKV_OK ? s.pending_offload : 0;
  }

  // Tag backend: every resident token on the device pool and every persisted
  // host chunk is read back and checked (sim.cpp check_conservation)
  void check_conservation() const {
    static_assert(!kValue, "conservation check uses the tag backend");
    detail::check(mtkv_engine_check_conservation(e_));
  }

  std::string dump_page_map() const {  // sim.hpp:493
    char* p = mtkv_dump_page_map(e_, 1);
    std::string s(p);
    mtkv_free(p);
    return s;
  }

  mtkv_engine* handle() const { return e_; }  // pipelined submit / rankings (include/mtkv_b200.h)

 private:
  mtkv_run_report raw_report() const {
    mtkv_run_report x;
    detail::check(mtkv_report(e_, 1, &x));
    return x;
  }
  EngineOptions opts_;
  detail::ManagerView view_;
  mtkv_engine* e_ = nullptr;
  std::uint32_t vocab_ = 0;
  std::uint32_t cfg_pages_ = 0;
};

}  // namespace b200
}  // namespace mtkv
