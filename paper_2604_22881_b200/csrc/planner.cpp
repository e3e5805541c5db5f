// Host control plane (see planner.hpp). Reference semantics followed, by
// section: manager.cpp:74-139 (prepare_metadata), :55 (ensure_free),
// :141 (evict_user), :178-202 (commit/finish/persist/scratch);
// pipeline.cpp:25 / :78 (onload / offload schedule); sim.hpp:212 (process_due),
// :303 (trigger_offloads), :332-455 (process_batch accounting).
#include "planner.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "devctl.hpp"

namespace mtkv_b200 {

static uint64_t div_up(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

Planner::Planner(const mtkv_kv_config& kv, const mtkv_cost_model& cost, int mode, bool keep_tokens)
    : kv_(kv), cost_(cost), mode_(mode), keep_tokens_(keep_tokens) {
  free_.resize(kv.device_pages);
  for (uint32_t i = 0; i < kv.device_pages; ++i) free_[i] = kv.device_pages - 1 - i;
  chunk_bytes_u64_ = uint64_t(kv.chunk_size) * uint64_t(kv.num_layers) * 2 * kv.num_heads *
                     kv.head_dim * kv.bytes_per_element;
  const uint64_t token_bytes = uint64_t(kv.num_layers) * 2 * kv.num_heads * kv.head_dim *
                               kv.bytes_per_element;
  chunk_bytes_ = double(kv.chunk_size) * double(token_bytes);
}

int Planner::slot_of(uint32_t id, bool create) {
  auto it = index_.find(id);
  if (it != index_.end()) return it->second;
  if (!create) return -1;
  int s = int(users_.size());
  users_.emplace_back();
  users_.back().id = id;
  index_.emplace(id, s);
  return s;
}

const UserRec* Planner::find(uint32_t user) const {
  auto it = index_.find(user);
  return it == index_.end() ? nullptr : &users_[it->second];
}

void Planner::lru_unlink(int s) {
  UserRec& u = users_[s];
  if (!u.in_lru) return;
  if (u.newer >= 0) users_[u.newer].older = u.older; else newest_ = u.older;
  if (u.older >= 0) users_[u.older].newer = u.newer; else oldest_ = u.newer;
  u.newer = u.older = -1;
  u.in_lru = false;
}

void Planner::lru_front(int s) {
  lru_unlink(s);
  UserRec& u = users_[s];
  u.older = newest_;
  if (newest_ >= 0) users_[newest_].newer = s; else oldest_ = s;
  newest_ = s;
  u.in_lru = true;
}

uint32_t Planner::pop_page() {
  uint32_t p = free_.back();
  free_.pop_back();
  ++occupied_;
  ++pages_allocated_;
  return p;
}

void Planner::push_page(uint32_t p) {
  if (!ctl_) free_.push_back(p);  // device mode: the free stack lives on the GPU
  --occupied_;
}

bool Planner::evict_slot(int s, uint64_t* freed, std::string& err) {
  UserRec& u = users_[s];
  if (u.locked) { err = "evict: user is locked"; return false; }
  if (!u.known) { err = "evict: unknown user"; return false; }
  uint64_t n = 0;
  if (u.has_pages) {
    n = u.pages.size();
    for (uint32_t p : u.pages) push_page(p);  // zero-copy: metadata only
    u.pages.clear();
    u.has_pages = false;
  }
  if (u.device_len > u.persisted_len) tail_lost_ += u.device_len - u.persisted_len;
  u.device_len = 0;
  ++evictions_;
  lru_unlink(s);
  if (freed) *freed = n;
  return true;
}

int Planner::evict(uint32_t user, std::string& err) {
  if (ctl_) { err = "evict: not available with the device planner (device tables own the pages)"; return MTKV_ERROR; }
  int s = slot_of(user, false);
  if (s < 0) { err = "evict: unknown user"; return MTKV_ERROR; }
  return evict_slot(s, nullptr, err) ? MTKV_OK : MTKV_ERROR;
}

int Planner::free_pages_for(uint64_t need, const std::vector<char>& in_batch, BatchWork& w) {
  while (free_.size() < need) {
    int v = oldest_;
    while (v >= 0 && (in_batch[v] || users_[v].locked)) v = users_[v].newer;
    if (v < 0) {
      w.error = "allocation unsatisfiable: all resident users locked or in batch";
      return MTKV_BATCH_REJECTED;
    }
    UserRec& u = users_[v];
    mtkv_eviction rec{u.id, 0, u.device_len > u.persisted_len ? u.device_len - u.persisted_len : 0};
    std::string err;
    evict_slot(v, &rec.freed_pages, err);
    w.evictions.push_back(rec);
  }
  return MTKV_OK;
}

void Planner::fire_completions(double now, std::vector<uint64_t>* persisted, BatchWork* w) {
  while (!pending_.empty() && pending_.top().done <= now) {
    Pending p = pending_.top();
    pending_.pop();
    UserRec& u = users_[p.slot];
    if (p.chunk_index != u.host_chunks.size()) {
      if (w) { w->rc = MTKV_ERROR; w->error = "host write: gap in chunk sequence"; }
      return;
    }
    if (kv_.host_capacity != 0 && host_total_ >= kv_.host_capacity) {
      if (w) { w->rc = MTKV_ERROR; w->error = "host write: capacity exceeded"; }
      return;
    }
    u.host_chunks.push_back(p.chunk_id);
    ++host_total_;
    u.persisted_len += kv_.chunk_size;
    quota_used_ -= kv_.chunk_size;
    if (--u.pending == 0) u.locked = false;
    note_update(p.slot);
    if (persisted) persisted->push_back(p.chunk_id);
  }
}

void Planner::drain(std::vector<uint64_t>* persisted) { fire_completions(1e300, persisted, nullptr); }

void Planner::schedule_onload(double submit, size_t n_chunks, std::vector<double>& fire) {
  const uint32_t L = kv_.num_layers;
  fire.assign(L, submit);
  if (n_chunks == 0) return;
  const double fill = chunk_bytes_ / cost_.host_bandwidth;
  const double dma = cost_.tx_setup + chunk_bytes_ / cost_.bus_bandwidth;
  const double scat = double(kv_.chunk_size / kv_.page_size) * cost_.page_op;
  for (size_t c = 0; c < n_chunks; ++c) {
    const uint64_t b = pinned_turn_++ % 2;
    const double fill_end = std::max({host_cpu_free_, pinned_free_[b], submit}) + fill;
    host_cpu_free_ = fill_end;
    const double dma_end = std::max(h2d_free_, fill_end) + dma;
    h2d_free_ = dma_end;
    pinned_free_[b] = dma_end;
    for (uint32_t l = 0; l < L; ++l) {
      const double s_end = std::max(scatter_free_, dma_end) + scat;
      scatter_free_ = s_end;
      fire[l] = std::max(fire[l], s_end);
    }
  }
  for (uint32_t l = 1; l < L; ++l) fire[l] = std::max(fire[l], fire[l - 1]);
}

double Planner::schedule_offload(double submit) {
  const double gather = double(kv_.num_layers) * double(kv_.chunk_size / kv_.page_size) * cost_.page_op;
  const double dma = cost_.tx_setup + chunk_bytes_ / cost_.bus_bandwidth;
  const double copy = chunk_bytes_ / cost_.host_bandwidth;
  const double gather_end = std::max(offload_free_, submit) + gather;
  const double dma_end = gather_end + dma;
  offload_free_ = dma_end;
  return dma_end + copy;
}

void Planner::trigger_offloads(int s, double t, BatchWork& w) {
  const uint64_t C = kv_.chunk_size;
  const uint32_t ppc = pages_per_chunk();
  for (;;) {
    UserRec& u = users_[s];
    const uint64_t covered = u.persisted_len + uint64_t(u.pending) * C;
    if (u.device_len < covered + C) break;
    if (quota_used_ + C > kv_.offload_quota) break;  // rejected; retried at the next append
    quota_used_ += C;
    const uint64_t ci = covered / C;
    ChunkMove m;
    m.chunk_id = next_chunk_id_++;
    m.user = u.id;
    m.chunk_index = uint32_t(ci);
    m.pages_off = uint32_t(w.pages.size());
    w.pages.insert(w.pages.end(), u.pages.begin() + ci * ppc, u.pages.begin() + (ci + 1) * ppc);
    w.offloads.push_back(m);
    const double done = schedule_offload(t);
    if (u.pending == 0) u.locked = true;
    ++u.pending;
    note_update(s);
    pending_.push(Pending{done, order_++, s, ci, m.chunk_id});
  }
}

// prepare_metadata (manager.cpp:74): touch + LRU, hit class, page growth and
// candidate scratch with ensure_free's evictions (manager.cpp:55), in request
// order; a repeated user plans against its earlier occurrence's projection.
bool Planner::prepare_metadata(const mtkv_request* reqs, uint32_t n, bool hier, std::vector<int>& slot,
                               std::vector<uint32_t>& scratch_ids, BatchWork& w) {
  for (uint32_t i = 0; i < n; ++i) slot[i] = slot_of(reqs[i].user, true);
  std::vector<char> in_batch(users_.size(), 0);
  for (uint32_t i = 0; i < n; ++i) in_batch[slot[i]] = 1;
  // projected (total_len, device_len) per distinct user, in request order
  std::unordered_map<int, std::pair<uint64_t, uint64_t>> proj;
  uint64_t batch_need = 0;
  for (uint32_t i = 0; i < n; ++i) {
    UserRec& u = users_[slot[i]];
    u.known = true;
    u.last_access = ++stamp_;
    lru_front(slot[i]);
    auto pit = proj.try_emplace(slot[i], u.total_len, u.device_len).first;
    const uint64_t prior = pit->second.first, devlen = pit->second.second;
    mtkv_request_plan& p = w.reqs[i].plan;
    p = mtkv_request_plan{};
    p.user = reqs[i].user;
    p.history_len = prior;
    p.delta = reqs[i].new_token_count;
    p.num_candidates = reqs[i].candidate_count;
    if (p.num_candidates < 1) {
      w.rc = MTKV_ERROR;
      w.error = "request: need at least one candidate";
      return false;
    }
    if (devlen > 0) {
      p.device_served = std::min(devlen, prior);
      p.reusable_len = p.device_served;
    } else if (hier && u.persisted_len > 0) {
      p.host_onload = u.persisted_len;
      p.reusable_len = u.persisted_len;
      p.onload_chunks = uint32_t(u.persisted_len / kv_.chunk_size);
    }
    p.fresh_history = prior - p.reusable_len;
    const uint64_t target = prior + p.delta;
    const uint64_t want = div_up(target, kv_.page_size);
    const uint64_t have = u.has_pages ? u.pages.size() : 0;
    const uint64_t grow = want > have ? want - have : 0;
    const uint64_t scratch = div_up(p.num_candidates, kv_.page_size);
    batch_need += grow + scratch;
    if (batch_need > kv_.device_pages) {
      w.rc = MTKV_BATCH_REJECTED;
      w.error = "batch exceeds total device pages";
      return false;
    }
    w.rc = free_pages_for(grow + scratch, in_batch, w);
    if (w.rc) return false;
    UserRec& uu = users_[slot[i]];
    uu.has_pages = true;
    for (uint64_t g = 0; g < grow; ++g) uu.pages.push_back(pop_page());
    w.reqs[i].scratch_off = uint32_t(scratch_ids.size());
    w.reqs[i].n_scratch = uint32_t(scratch);
    for (uint64_t g = 0; g < scratch; ++g) scratch_ids.push_back(pop_page());
    p.scratch_pages = uint32_t(scratch);
    pit->second = {target, p.reusable_len + p.fresh_history + p.delta};
  }
  return true;
}

// ---- CacheManager step surface (manager.hpp:89-147): prepare_metadata and the
// calls Engine<B>::process_batch makes after it, one at a time, for callers that
// drive the manager themselves (the reference's manager tests do).
int Planner::mgr_prepare(const mtkv_request* reqs, uint32_t n, bool host_enabled, std::string& err) {
  BatchWork w;
  w.reqs.resize(n);
  std::vector<int> slot(n);
  std::vector<uint32_t> ids;
  const bool ok = prepare_metadata(reqs, n, host_enabled, slot, ids, w);
  if (!ok && w.rc == MTKV_BATCH_REJECTED) {  // the reference keeps what happened before the throw
    err = w.error;
    last_ = w;
    last_.reqs.clear();
    return MTKV_BATCH_REJECTED;
  }
  if (!ok) { err = w.error; return w.rc ? w.rc : MTKV_ERROR; }
  mgr_scratch_.assign(n, {});
  for (uint32_t i = 0; i < n; ++i) {
    w.reqs[i].slot = uint32_t(slot[i]);
    mgr_scratch_[i].assign(ids.begin() + w.reqs[i].scratch_off, ids.begin() + w.reqs[i].scratch_off + w.reqs[i].n_scratch);
  }
  last_ = w;
  return MTKV_OK;
}

const std::vector<uint32_t>* Planner::mgr_scratch(uint32_t i) const {
  return i < mgr_scratch_.size() ? &mgr_scratch_[i] : nullptr;
}

int Planner::mgr_release_pages(const uint32_t* pages, uint32_t n, std::string& err) {
  for (uint32_t i = 0; i < n; ++i) {  // alloc_.release (store.hpp:76) of each scratch page
    if (pages[i] >= kv_.device_pages) { err = "device store: releasing free page"; return MTKV_ERROR; }
    push_page(pages[i]);
  }
  return MTKV_OK;
}

int Planner::mgr_commit_onload(uint32_t user, uint64_t reusable_len, uint32_t onload_chunks, std::string& err) {
  if (onload_chunks == 0) return MTKV_OK;  // manager.cpp:179 no pending onload: no-op
  const int s = slot_of(user, false);
  if (s < 0 || !users_[s].known) { err = "commit_onload: unknown user"; return MTKV_ERROR; }
  users_[s].device_len = reusable_len;
  return MTKV_OK;
}

int Planner::mgr_finish_append(uint32_t user, uint64_t appended, std::string& err) {
  const int s = slot_of(user, false);
  if (s < 0 || !users_[s].known) { err = "finish_append: unknown user"; return MTKV_ERROR; }
  UserRec& u = users_[s];
  u.device_len += appended;
  u.total_len = std::max(u.total_len, u.device_len);
  return MTKV_OK;
}

int Planner::mgr_advance_persisted(uint32_t user, uint64_t tokens, std::string& err) {
  const int s = slot_of(user, false);
  if (s < 0 || !users_[s].known) { err = "advance_persisted: unknown user"; return MTKV_ERROR; }
  UserRec& u = users_[s];
  u.persisted_len += tokens;
  if (u.persisted_len > u.total_len) { err = "persist: beyond total length"; return MTKV_ERROR; }
  return MTKV_OK;
}

int Planner::mgr_lock(uint32_t user, bool lock, std::string& err) {
  const int s = slot_of(user, false);
  if (lock) {
    if (s < 0 || !users_[s].known) { err = "lock: unknown user"; return MTKV_ERROR; }
    if (users_[s].locked) { err = "lock: user already locked"; return MTKV_ERROR; }
  } else if (s < 0 || !users_[s].locked) {
    err = "unlock: user not locked";
    return MTKV_ERROR;
  }
  users_[s].locked = lock;
  return MTKV_OK;
}

uint32_t Planner::last_page_len(uint32_t user) const {
  const UserRec* u = find(user);
  if (!u || u->device_len == 0) return 0;
  const uint32_t rem = uint32_t(u->device_len % kv_.page_size);
  return rem == 0 ? kv_.page_size : rem;
}

// Adaptive onload policy. Split form (default): every host hit re-encodes the
// same fraction f of its persisted chunks — its EARLIEST chunks, whose
// positions attend over the fewest keys, so a re-encoded token costs the SMs
// less than one late in the history — and onloads the rest; f balances the
// batch's SM time (fresh rows + re-encoded rows at recompute_tps_) against its
// host-link time (onloaded chunks at link_Bps_). The positions a request
// re-encodes are [0, f n C): disjoint from its own fresh rows, so the executor
// runs them as an extra request (BatchWork keeps one ReqWork per request).
// Whole form (MTKV_ADAPTIVE_SPLIT=0): walk the host hits and send each whole
// prefix to whichever resource would finish it earlier.
void Planner::choose_recompute(BatchWork& w) {
  static const bool split = [] {
    const char* e = std::getenv("MTKV_ADAPTIVE_SPLIT");
    return !(e && e[0] == '0');
  }();
  double t_sm = 0;
  for (const ReqWork& r : w.reqs)
    t_sm += double(r.plan.fresh_history + r.plan.delta + r.plan.num_candidates) / recompute_tps_;
  const double c_link_chunk = double(chunk_bytes_u64_) / link_Bps_, c_sm_chunk = double(kv_.chunk_size) / recompute_tps_;
  if (split) {
    double chunks = 0;
    for (const ReqWork& r : w.reqs) chunks += r.plan.onload_chunks;
    if (chunks == 0) return;
    // t_sm + f * chunks * c_sm = (1 - f) * chunks * c_link
    const double f = std::min(1.0, std::max(0.0, (chunks * c_link_chunk - t_sm) / (chunks * (c_link_chunk + c_sm_chunk))));
    for (ReqWork& r : w.reqs) {
      const uint32_t n = r.plan.onload_chunks;
      if (!n) continue;
      const uint32_t k = std::min<uint32_t>(n, uint32_t(std::lround(f * n)));
      if (k == n) r.recompute_prefix = true;  // contiguous with the request's own rows: one request
      else r.head_chunks = k;
    }
    return;
  }
  double t_link = 0;
  for (ReqWork& r : w.reqs) {
    if (!r.plan.onload_chunks) continue;
    const double c_link = double(r.plan.onload_chunks) * c_link_chunk;
    const double c_sm = double(r.plan.reusable_len) / recompute_tps_;
    if (t_link + c_link <= t_sm + c_sm) {
      t_link += c_link;
    } else {
      r.recompute_prefix = true;
      t_sm += c_sm;
    }
  }
}

void Planner::plan_batch(const mtkv_request* reqs, uint32_t n, BatchWork& w) {
  w = BatchWork();
  if (n == 0) return;
  const bool hier = mode_ == MTKV_MODE_HIERARCHICAL;
  const bool cached = mode_ != MTKV_MODE_RECOMPUTE;
  const double start = clock_;
  w.sim_start = start;
  fire_completions(start, &w.persisted, &w);
  if (w.rc) return;
  double t = start, st[9] = {0};
  std::vector<int> slot(n);
  w.reqs.resize(n);
  std::vector<uint32_t> scratch_ids;

  if (cached && ctl_) {
    if (!prepare_on_device(reqs, n, slot, scratch_ids, w)) return;
    st[0] = cost_.meta_fixed;
  } else if (cached) {
    if (!prepare_metadata(reqs, n, hier, slot, scratch_ids, w)) return;
    st[0] = cost_.meta_fixed;
  } else {
    for (uint32_t i = 0; i < n; ++i) {
      slot[i] = slot_of(reqs[i].user, true);
      UserRec& u = users_[slot[i]];
      mtkv_request_plan& p = w.reqs[i].plan;
      p = mtkv_request_plan{};
      p.user = reqs[i].user;
      p.history_len = u.recompute_len;
      p.delta = reqs[i].new_token_count;
      p.num_candidates = reqs[i].candidate_count;
      p.fresh_history = p.history_len;
      u.recompute_len += p.delta;
    }
  }
  peak_pages_ = std::max(peak_pages_, occupied_);
  t += st[0];

  // Onload plan in the reference's staging order (sim.hpp:371-383).
  size_t total_chunks = 0;
  for (uint32_t i = 0; i < n; ++i) total_chunks += w.reqs[i].plan.onload_chunks;
  std::vector<double> fire;
  schedule_onload(t, total_chunks, fire);
  if (uint64_t(total_chunks) * kv_.chunk_size > uint64_t(kv_.onload_pages) * kv_.page_size) {
    w.rc = MTKV_ERROR;
    w.error = "onload buffer: batch exceeds staging capacity";
    return;
  }

  // Snapshot page tables after allocation (a user's later occurrences in this
  // batch grew the same list) and lay out the executor's work.
  const uint32_t ppc = pages_per_chunk();
  for (uint32_t i = 0; i < n; ++i) {
    ReqWork& r = w.reqs[i];
    r.slot = uint32_t(slot[i]);
    if (cached) {
      const UserRec& u = users_[slot[i]];
      r.pages_off = uint32_t(w.pages.size());
      r.n_pages = uint32_t(u.pages.size());
      w.pages.insert(w.pages.end(), u.pages.begin(), u.pages.end());
    }
  }
  for (uint32_t i = 0; i < n; ++i) {
    ReqWork& r = w.reqs[i];
    const uint32_t so = uint32_t(w.pages.size());
    w.pages.insert(w.pages.end(), scratch_ids.begin() + r.scratch_off,
                   scratch_ids.begin() + r.scratch_off + r.n_scratch);
    r.scratch_off = so;
  }
  if (hier && policy_ == MTKV_ONLOAD_ADAPTIVE) choose_recompute(w);
  for (uint32_t i = 0; i < n; ++i) {
    const ReqWork& r = w.reqs[i];
    const UserRec& u = users_[slot[i]];
    if (r.plan.onload_chunks) {
      const uint64_t head = r.recompute_prefix ? r.plan.reusable_len : uint64_t(r.head_chunks) * kv_.chunk_size;
      prefix_recomputed_ += head;
      prefix_onloaded_ += r.plan.reusable_len - head;
    }
    if (r.recompute_prefix) continue;  // its K/V is re-encoded, nothing crosses the host link
    for (uint32_t c = r.head_chunks; c < r.plan.onload_chunks; ++c) {  // the re-encoded head is not onloaded
      ChunkMove m;
      m.chunk_id = u.host_chunks[c];
      m.user = u.id;
      m.chunk_index = c;
      m.pages_off = r.pages_off + c * ppc;
      w.onloads.push_back(m);
    }
  }

  uint64_t fresh_total = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const auto& p = w.reqs[i].plan;
    fresh_total += p.fresh_history + p.delta + p.num_candidates;
  }
  if (cached) st[1] = cost_.strip_fixed;
  st[2] = cost_.embed_fixed + cost_.embed_coeff * double(fresh_total);
  st[3] = cost_.layout_fixed + cost_.layout_coeff * double(fresh_total);
  if (cached) {
    st[4] = cost_.await_fixed;
    st[5] = cost_.update_fixed + cost_.commit_per_chunk * double(total_chunks);
  }
  t += st[1] + st[2] + st[3] + st[4] + st[5];

  if (cached)  // commit_onload (manager.cpp:178)
    for (uint32_t i = 0; i < n; ++i)
      if (w.reqs[i].plan.onload_chunks > 0) users_[slot[i]].device_len = w.reqs[i].plan.reusable_len;

  double dominant = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const auto& p = w.reqs[i].plan;
    const double fresh = double(p.fresh_history + p.delta + p.num_candidates);
    const double total = double(p.history_len + p.delta + p.num_candidates);
    dominant = std::max(dominant, cost_.attn_coeff * fresh * total + cost_.linear_coeff * fresh);
  }
  const double layer_comp = double(n) * dominant;
  for (uint32_t l = 0; l < kv_.num_layers; ++l) {
    const double wait = std::max(0.0, fire[l] - t);
    t += wait;
    wait_ += wait;
    t += layer_comp;
    comp_ += layer_comp;
    st[6] += wait + layer_comp;
  }

  // Encode bookkeeping in request order (sim.hpp:246 encode_and_append).
  for (uint32_t i = 0; i < n; ++i) {
    ReqWork& r = w.reqs[i];
    UserRec& u = users_[slot[i]];
    const auto& p = r.plan;
    if (r.head_chunks) {  // split host hit: the re-encoded head's token ids (positions [0, head_rows))
      r.head_rows = r.head_chunks * kv_.chunk_size;
      r.head_tok_off = uint32_t(w.tokens.size());
      if (keep_tokens_) {
        if (u.tokens.size() < r.head_rows) {
          w.rc = MTKV_ERROR;
          w.error = "value mode: trace must carry explicit token ids";
          return;
        }
        w.tokens.insert(w.tokens.end(), u.tokens.begin(), u.tokens.begin() + r.head_rows);
      }
      w.fresh_rows += r.head_rows;
    }
    r.tok_off = uint32_t(w.tokens.size());
    if (cached) {
      // a re-encoded host-hit prefix (adaptive policy) is appended from position 0
      const uint64_t from = r.recompute_prefix ? 0 : p.reusable_len;
      r.start = r.recompute_prefix ? 0 : u.device_len;
      r.n_hist = uint32_t(p.fresh_history + p.delta + (p.reusable_len - from));
      if (keep_tokens_) {
        if (u.tokens.size() != p.history_len) {
          w.rc = MTKV_ERROR;
          w.error = "value mode: trace must carry explicit token ids";
          return;
        }
        w.tokens.insert(w.tokens.end(), u.tokens.begin() + from, u.tokens.end());
      }
      u.device_len += p.fresh_history + p.delta;  // finish_append (manager.cpp:184)
      u.total_len = std::max(u.total_len, u.device_len);
    } else {
      r.start = 0;
      r.n_hist = uint32_t(p.history_len + p.delta);
      if (keep_tokens_) w.tokens.insert(w.tokens.end(), u.tokens.begin(), u.tokens.end());
    }
    if (keep_tokens_) {
      if (reqs[i].new_tokens) {
        w.tokens.insert(w.tokens.end(), reqs[i].new_tokens, reqs[i].new_tokens + reqs[i].new_token_count);
        u.tokens.insert(u.tokens.end(), reqs[i].new_tokens, reqs[i].new_tokens + reqs[i].new_token_count);
      }
      if (reqs[i].candidates)
        w.tokens.insert(w.tokens.end(), reqs[i].candidates, reqs[i].candidates + reqs[i].candidate_count);
    }
    w.fresh_rows += r.n_hist + p.num_candidates;
  }

  if (cached)  // release_scratch (manager.cpp:196), request order
    for (uint32_t id : scratch_ids) push_page(id);

  if (hier) {
    st[7] = cost_.offload_submit;
    for (uint32_t i = 0; i < n; ++i) trigger_offloads(slot[i], t, w);
    t += st[7];
  }
  st[8] = cost_.post_fixed;
  t += st[8];

  clock_ = t;
  w.sim_end = t;
  latency_ += t - start;
  for (int i = 0; i < 9; ++i) steps_[i] += st[i];
  ++batches_;
  requests_ += n;
  for (uint32_t i = 0; i < n; ++i) {
    const auto& p = w.reqs[i].plan;
    if (p.history_len > 0) {
      required_ += p.history_len;
      dev_served_ += p.device_served;
      host_served_ += p.host_onload;
    }
    processed_ += p.fresh_history + p.delta + p.num_candidates;
  }
}

void Planner::note_update(int s) {
  if (!ctl_) return;
  const UserRec& u = users_[s];
  const CtlUpd c{uint32_t(s), u.locked ? 1u : 0u, u.persisted_len};
  auto it = ctl_upd_at_.find(s);
  if (it != ctl_upd_at_.end()) ctl_upd_[it->second] = c;  // absolute values: latest wins
  else {
    ctl_upd_at_.emplace(s, ctl_upd_.size());
    ctl_upd_.push_back(c);
  }
}

// prepare_metadata (manager.cpp:74) with the decisions taken on the GPU: the
// mirror applies slots, touches, evictions and page ids exactly as returned.
bool Planner::prepare_on_device(const mtkv_request* reqs, uint32_t n, std::vector<int>& slot,
                                std::vector<uint32_t>& scratch_ids, BatchWork& w) {
  std::vector<CtlReq> cr(n);
  for (uint32_t i = 0; i < n; ++i) cr[i] = CtlReq{reqs[i].user, reqs[i].new_token_count, reqs[i].candidate_count, 0};
  std::string err;
  const int rc = ctl_->prepare(cr.data(), n, ctl_upd_, err);
  ctl_upd_.clear();
  ctl_upd_at_.clear();
  if (rc) {
    w.rc = MTKV_ERROR;
    w.error = err;
    return false;
  }
  const CtlHdr& h = ctl_->hdr();
  const CtlPlan* pl = ctl_->plans();
  for (uint32_t i = 0; i < n; ++i) {
    slot[i] = slot_of(reqs[i].user, true);
    if (i < uint32_t(h.fail_at) && pl[i].slot != slot[i]) {
      w.rc = MTKV_ERROR;
      w.error = "device planner: slot numbering diverged from the host mirror";
      return false;
    }
  }
  const uint32_t touched = h.fail == CTL_OK ? n : uint32_t(h.fail_at) + 1;
  for (uint32_t i = 0; i < touched && i < n; ++i) {
    UserRec& u = users_[slot[i]];
    u.known = true;
    u.last_access = ++stamp_;
    lru_front(slot[i]);
  }
  for (uint32_t e = 0; e < h.n_evict; ++e) {  // zero-copy evictions, in the device's order
    const CtlEvict& ev = ctl_->evictions()[e];
    UserRec& v = users_[ev.slot];
    w.evictions.push_back(mtkv_eviction{v.id, ev.freed_pages, ev.tail_lost});
    occupied_ -= v.pages.size();
    v.pages.clear();
    v.has_pages = false;
    if (v.device_len > v.persisted_len) tail_lost_ += v.device_len - v.persisted_len;
    v.device_len = 0;
    ++evictions_;
    lru_unlink(int(ev.slot));
  }
  const uint32_t allocated = std::min<uint32_t>(n, uint32_t(h.fail_at));
  const uint32_t* ids = ctl_->ids();
  for (uint32_t i = 0; i < allocated; ++i) {
    const CtlPlan& c = pl[i];
    mtkv_request_plan& p = w.reqs[i].plan;
    p = mtkv_request_plan{};
    p.user = reqs[i].user;
    p.history_len = c.history_len;
    p.delta = reqs[i].new_token_count;
    p.num_candidates = reqs[i].candidate_count;
    p.device_served = c.device_served;
    p.host_onload = c.host_onload;
    p.reusable_len = c.reusable_len;
    p.onload_chunks = c.onload_chunks;
    p.fresh_history = c.fresh_history;
    UserRec& u = users_[slot[i]];
    u.has_pages = true;
    u.pages.insert(u.pages.end(), ids + c.grow_off, ids + c.grow_off + c.grow_n);
    w.reqs[i].scratch_off = uint32_t(scratch_ids.size());
    w.reqs[i].n_scratch = c.scratch_n;
    scratch_ids.insert(scratch_ids.end(), ids + c.scratch_off, ids + c.scratch_off + c.scratch_n);
    p.scratch_pages = c.scratch_n;
    occupied_ += c.grow_n + c.scratch_n;
    pages_allocated_ += c.grow_n + c.scratch_n;
  }
  if (h.fail != CTL_OK) {
    if (h.fail == CTL_BAD_REQUEST) {
      w.rc = MTKV_ERROR;
      w.error = "request: need at least one candidate";
    } else {
      w.rc = MTKV_BATCH_REJECTED;
      w.error = h.fail == CTL_REJECT_PAGES ? "batch exceeds total device pages"
                                           : "allocation unsatisfiable: all resident users locked or in batch";
    }
    return false;
  }
  return true;
}

std::vector<uint32_t> Planner::known_users() const {
  std::vector<uint32_t> out;
  for (const auto& u : users_)
    if (u.known) out.push_back(u.id);
  std::sort(out.begin(), out.end());
  return out;
}

std::vector<uint32_t> Planner::lru_snapshot() const {
  std::vector<uint32_t> out;
  for (int s = newest_; s >= 0; s = users_[s].older) out.push_back(users_[s].id);
  return out;
}

void Planner::report(mtkv_run_report& r) const {
  std::memset(&r, 0, sizeof(r));
  const double nb = batches_ ? double(batches_) : 1.0;
  for (int i = 0; i < 9; ++i) r.step_ms[i] = steps_[i] / nb * 1e3;
  r.wait_ms = wait_ / nb * 1e3;
  r.comp_ms = comp_ / nb * 1e3;
  if (required_ == 0) {
    r.gpu_hit_ratio = r.total_hit_ratio = 1.0;
  } else {
    r.gpu_hit_ratio = double(dev_served_) / double(required_);
    r.total_hit_ratio = double(dev_served_ + host_served_) / double(required_);
  }
  r.tokens_processed = processed_;
  r.evictions = evictions_;
  r.tail_tokens_lost = tail_lost_;
  r.requests = requests_;
  r.batches = batches_;
  r.avg_latency_ms = latency_ / nb * 1e3;
  r.total_latency_ms = latency_ * 1e3;
  r.peak_pages = peak_pages_;
  r.pages_allocated = pages_allocated_;
  r.occupied_pages = occupied_;
  r.free_pages = kv_.device_pages - occupied_;
  r.quota_in_flight = quota_used_;
  r.clock = clock_;
  r.hist_required = required_;
  r.hist_device = dev_served_;
  r.hist_host = host_served_;
  r.prefix_onloaded = prefix_onloaded_;
  r.prefix_recomputed = prefix_recomputed_;
}

}  // namespace mtkv_b200
