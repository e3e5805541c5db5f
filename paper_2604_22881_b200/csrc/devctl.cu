// Device-side control plane (see devctl.hpp for the design and the reference
// functions it restates). One CTA of 512 threads per batch.
#include "devctl.hpp"

#include <algorithm>
#include <cstring>

namespace mtkv_b200 {

namespace {

constexpr int kThreads = 512;
constexpr uint32_t kMaxVictims = 4096;  // per batch (bitonic sort in shared memory)
constexpr uint32_t F_KNOWN = 1, F_HAS_PAGES = 2, F_LOCKED = 4, F_IN_LRU = 8;
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

struct Globals {
  uint32_t top, n_slots, epoch, pad;
  uint64_t stamp;
};

struct State {  // device tables (one allocation)
  Globals* g;
  uint32_t *keys, *vals;                  // hash: user id -> slot
  uint64_t *total, *dev, *pers, *last;    // per slot
  uint32_t *flags, *npages, *mark, *firsti;
  uint32_t* ptab;                         // [max_users][max_pages]
  uint32_t* stack;                        // free page ids, stack[top-1] handed out next
};

struct Args {
  State s;
  const CtlReq* reqs;
  uint32_t n;
  const CtlUpd* upd;
  uint32_t n_upd;
  CtlHdr* hdr;
  CtlPlan* plans;
  CtlEvict* evict;
  uint32_t* ids;
  uint32_t device_pages, page_size, chunk_size, max_users, max_pages, hash_mask;
  uint32_t hier;
  uint64_t staging_tokens;  // onload staging capacity (KVConfig::onload_pages * page_size)
};

__device__ __forceinline__ uint32_t hash_u32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ uint64_t div_up(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// shared-memory working set (dynamic: per-request arrays follow)
struct Smem {
  uint64_t w_hist[256];   // radix-select weights per digit
  uint32_t c_hist[256];
  uint64_t red64[kThreads / 32];
  uint32_t red32[kThreads / 32];
  uint64_t prefix, need, wtotal;
  uint32_t prefix_bits, n_vict, fail, fail_at, i_end, n_ids, n_ev, top;
  uint64_t vkey[kMaxVictims];   // (stamp) of each victim
  uint32_t vslot[kMaxVictims];
  uint32_t vnp[kMaxVictims];    // pages a victim frees
  uint32_t vpos[kMaxVictims];   // stack position its first page is pushed to
  uint32_t vreq[kMaxVictims];   // request whose ensure_free evicted it
  uint32_t min_pos, max_pos, final_top, scratch_total, old_slots;
};

__device__ uint64_t block_sum64(uint64_t v, Smem& sm) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) sm.red64[w] = v;
  __syncthreads();
  uint64_t t = 0;
  for (int i = 0; i < kThreads / 32; ++i) t += sm.red64[i];
  __syncthreads();
  return t;
}

// A batch the device tables cannot hold (CTL_CAPACITY) or the staging buffer
// cannot onload (CTL_STAGING) fails before any state changes except step 1's
// new users: remove their hash entries again. With linear probing this is
// exact because every key inserted by this batch is removed (older keys never
// probed through those positions: they were empty when the older keys went in).
__device__ void rollback_inserts(const Args& a, const uint32_t* r_slot, uint32_t old_slots, int32_t fail) {
  const State& S = a.s;
  for (uint32_t i = 0; i < a.n; ++i) {
    if (r_slot[i] < old_slots || r_slot[i] == kEmpty) continue;
    const uint32_t user = a.reqs[i].user;
    for (uint32_t h = hash_u32(user) & a.hash_mask;; h = (h + 1) & a.hash_mask) {
      const uint32_t k = S.keys[h];
      if (k == kEmpty) break;
      if (k == user) { S.keys[h] = kEmpty; break; }
    }
  }
  S.g->n_slots = old_slots;
  CtlHdr h{};
  h.fail = fail;
  h.fail_at = 0;
  h.n_slots = old_slots;
  *a.hdr = h;
}

__global__ void __launch_bounds__(kThreads, 1) ctl_prepare_kernel(Args a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  uint32_t* r_slot = reinterpret_cast<uint32_t*>(smem_raw + sizeof(Smem));
  uint32_t* r_grow = r_slot + a.n;
  uint32_t* r_scr = r_grow + a.n;
  uint64_t* r_cum = reinterpret_cast<uint64_t*>(r_scr + a.n + (a.n & 1));  // cumulative pages allocated
  uint64_t* p_total = r_cum + a.n;  // projections, kept at a user's first occurrence
  uint64_t* p_dev = p_total + a.n;
  uint64_t* p_have = p_dev + a.n;
  uint64_t* r_pers = p_have + a.n;   // persisted length (first occurrence)
  uint32_t* r_first = reinterpret_cast<uint32_t*>(r_pers + a.n);
  uint32_t* r_havei = r_first + a.n;  // pages the user holds before request i's grow
  uint32_t* r_pop = r_havei + a.n;    // stack position of request i's lowest popped page
  uint32_t* r_nv = r_pop + a.n;       // victims consumed up to and including request i
  uint32_t* r_ids = r_nv + a.n;       // grow ids offset of request i
  const uint32_t tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  State& S = a.s;
  Globals& G = *S.g;

  // ---- 0. host-side changes since the last batch (persist completions, offload locks) ----
  for (uint32_t i = tid; i < a.n_upd; i += kThreads) {
    const CtlUpd u = a.upd[i];
    S.pers[u.slot] = u.persisted_len;
    S.flags[u.slot] = u.locked ? (S.flags[u.slot] | F_LOCKED) : (S.flags[u.slot] & ~F_LOCKED);
  }
  if (tid == 0) {
    sm.fail = CTL_OK;
    sm.fail_at = a.n;
    sm.n_vict = 0;
    sm.old_slots = G.n_slots;
  }
  __syncthreads();

  // ---- 1. batched lookup / insert (warp 0): lane-parallel probing, ballot + match_any
  //         dedupe, new slots numbered in order of first appearance (manager.cpp:200) ----
  if (warp == 0) {
    uint32_t n_slots = G.n_slots;
    for (uint32_t base = 0; base < a.n; base += 32) {
      const uint32_t i = base + lane;
      const bool act = i < a.n;
      const uint32_t user = act ? a.reqs[i].user : 0;
      int32_t slot = -1;
      uint32_t h = hash_u32(user) & a.hash_mask;
      if (act) {
        for (;;) {
          const uint32_t k = S.keys[h];
          if (k == user) { slot = int32_t(S.vals[h]); break; }
          if (k == kEmpty) break;
          h = (h + 1) & a.hash_mask;
        }
      }
      const uint32_t miss = __ballot_sync(0xffffffffu, act && slot < 0);
      if (miss) {
        const uint32_t same = __match_any_sync(0xffffffffu, (act && slot < 0) ? user : kEmpty);
        const bool leader = act && slot < 0 && (__ffs(same) - 1) == int(lane);
        const uint32_t leaders = __ballot_sync(0xffffffffu, leader);
        int32_t mine = -1;
        if (leader) {
          mine = int32_t(n_slots + __popc(leaders & ((1u << lane) - 1)));
          if (uint32_t(mine) >= a.max_users) {
            sm.fail = CTL_CAPACITY;
          } else {
            for (;;) {  // insert (keys are distinct among leaders)
              const uint32_t prev = atomicCAS(&S.keys[h], kEmpty, user);
              if (prev == kEmpty || prev == user) break;
              h = (h + 1) & a.hash_mask;
            }
            S.vals[h] = uint32_t(mine);
            S.total[mine] = S.dev[mine] = S.pers[mine] = S.last[mine] = 0;
            S.flags[mine] = 0;
            S.npages[mine] = 0;
            S.mark[mine] = 0;
          }
        }
        const int src = __ffs(same) - 1;
        const int32_t got = __shfl_sync(0xffffffffu, mine, src);
        if (act && slot < 0) slot = got;
        n_slots += __popc(leaders);
        __threadfence_block();
      }
      if (act) r_slot[i] = slot < 0 ? kEmpty : uint32_t(slot);
      __syncwarp();
    }
    if (lane == 0) G.n_slots = min(n_slots, a.max_users);
  }
  __syncthreads();
  if (sm.fail == CTL_CAPACITY) {
    if (tid == 0) rollback_inserts(a, r_slot, sm.old_slots, CTL_CAPACITY);
    return;
  }
  const uint32_t epoch = G.epoch + 1;
  // ---- 2. batch membership, first occurrence, per-request state into shared memory ----
  for (uint32_t i = tid; i < a.n; i += kThreads) S.firsti[r_slot[i]] = 0xFFFFFFFFu;
  __syncthreads();
  for (uint32_t i = tid; i < a.n; i += kThreads) {
    S.mark[r_slot[i]] = epoch;
    atomicMin(&S.firsti[r_slot[i]], i);
  }
  __syncthreads();
  for (uint32_t i = tid; i < a.n; i += kThreads) {
    const uint32_t s = r_slot[i], f = S.firsti[s];
    r_first[i] = f;
    if (f == i) {
      p_total[i] = S.total[s];
      p_dev[i] = S.dev[s];
      p_have[i] = (S.flags[s] & F_HAS_PAGES) ? S.npages[s] : 0;
      r_pers[i] = S.pers[s];
    }
  }
  __syncthreads();

  // ---- 3. plan numbers in request order (thread 0, shared memory only; a repeated
  //         user plans against its earlier occurrence's projection, manager.cpp:91-137) ----
  if (tid == 0) {
    G.epoch = epoch;
    uint64_t batch_need = 0;
    uint32_t fail_at = a.n, fail = CTL_OK;
    for (uint32_t i = 0; i < a.n; ++i) {
      const uint32_t f = r_first[i];
      const uint64_t prior = p_total[f], devlen = p_dev[f], have = p_have[f], pers = r_pers[f];
      CtlPlan p{};
      p.slot = int32_t(r_slot[i]);
      p.history_len = prior;
      const uint32_t delta = a.reqs[i].delta, nc = a.reqs[i].ncand;
      if (nc < 1) { fail = CTL_BAD_REQUEST; fail_at = i; break; }
      if (devlen > 0) {
        p.device_served = devlen < prior ? devlen : prior;
        p.reusable_len = p.device_served;
      } else if (a.hier && pers > 0) {
        p.host_onload = pers;
        p.reusable_len = pers;
        p.onload_chunks = uint32_t(pers / a.chunk_size);
      }
      p.fresh_history = prior - p.reusable_len;
      const uint64_t target = prior + delta;
      const uint64_t want = div_up(target, a.page_size);
      const uint64_t grow = want > have ? want - have : 0;
      const uint64_t scratch = div_up(nc, a.page_size);
      batch_need += grow + scratch;
      if (batch_need > a.device_pages) { fail = CTL_REJECT_PAGES; fail_at = i; break; }
      if (have + grow > a.max_pages) { fail = CTL_CAPACITY; fail_at = i; break; }  // page-table row full
      r_grow[i] = uint32_t(grow);
      r_scr[i] = uint32_t(scratch);
      r_cum[i] = batch_need;
      r_havei[i] = uint32_t(have);
      a.plans[i] = p;
      p_total[f] = target;
      p_dev[f] = p.reusable_len + p.fresh_history + delta;
      p_have[f] = have + grow;
    }
    sm.fail = fail;
    sm.fail_at = fail_at;
  }
  __syncthreads();
  if (sm.fail == CTL_CAPACITY) {  // nothing but the step-1 inserts has changed yet
    if (tid == 0) rollback_inserts(a, r_slot, sm.old_slots, CTL_CAPACITY);
    return;
  }
  // ---- 4. eviction victims: oldest stamps among in-list, unlocked, not-in-batch users ----
  const uint32_t n_ok = sm.fail_at;  // requests whose allocation is attempted
  const uint64_t free0 = G.top;
  const uint32_t n_slots = G.n_slots;
  uint64_t wloc = 0;
  for (uint32_t s = tid; s < n_slots; s += kThreads) {
    const uint32_t f = S.flags[s];
    if ((f & F_IN_LRU) && !(f & F_LOCKED) && S.mark[s] != epoch) wloc += (f & F_HAS_PAGES) ? S.npages[s] : 0;
  }
  const uint64_t wtotal = block_sum64(wloc, sm);
  if (tid == 0) {
    // first request whose cumulative need cannot be covered even by evicting everyone
    uint32_t ex = n_ok;
    for (uint32_t i = 0; i < n_ok; ++i)
      if (r_cum[i] > free0 + wtotal) { ex = i; break; }
    sm.i_end = n_ok;
    if (ex < n_ok) {
      sm.fail = CTL_REJECT_VICTIMS;
      sm.fail_at = ex;
      sm.i_end = ex;
      sm.need = ~uint64_t(0);  // evict every eligible user
    } else {
      const uint64_t cum = n_ok ? r_cum[n_ok - 1] : 0;
      sm.need = cum > free0 ? cum - free0 : 0;
      if (sm.fail == CTL_OK && a.staging_tokens) {  // the onload staging check (sim.hpp:371) comes
        uint64_t tok = 0;                           // after a successful prepare_metadata
        for (uint32_t i = 0; i < n_ok; ++i) tok += uint64_t(a.plans[i].onload_chunks) * a.chunk_size;
        if (tok > a.staging_tokens) sm.fail = CTL_STAGING;
      }
    }
    sm.prefix = 0;
    sm.prefix_bits = 0;
  }
  __syncthreads();
  if (sm.fail == CTL_STAGING) {
    if (tid == 0) rollback_inserts(a, r_slot, sm.old_slots, CTL_STAGING);
    return;
  }
  const uint64_t need = sm.need;
  if (need > 0) {
    uint64_t thresh = ~uint64_t(0);
    if (need != ~uint64_t(0)) {
      // weighted radix select (8-bit digits, most significant first) of the stamp
      // threshold tau = min{t : pages(eligible, stamp <= t) >= need}; leading
      // all-zero digits of the largest stamp are skipped
      int top_shift = 0;
      for (uint64_t m = G.stamp >> 8; m; m >>= 8) top_shift += 8;
      uint64_t rem = need;
      for (int shift = top_shift; shift >= 0; shift -= 8) {
        for (uint32_t b = tid; b < 256; b += kThreads) { sm.w_hist[b] = 0; sm.c_hist[b] = 0; }
        __syncthreads();
        const uint64_t pre = sm.prefix;
        const int hi = shift + 8;  // bits above this digit fixed by the prefix
        for (uint32_t s = tid; s < n_slots; s += kThreads) {
          const uint32_t f = S.flags[s];
          if (!((f & F_IN_LRU) && !(f & F_LOCKED) && S.mark[s] != epoch)) continue;
          const uint64_t st = S.last[s];
          if (hi < 64 && (st >> hi) != (pre >> hi)) continue;
          const uint32_t dg = uint32_t(st >> shift) & 255u;
          atomicAdd(reinterpret_cast<unsigned long long*>(&sm.w_hist[dg]),
                    (unsigned long long)((f & F_HAS_PAGES) ? S.npages[s] : 0));
          atomicAdd(&sm.c_hist[dg], 1u);
        }
        __syncthreads();
        if (tid == 0) {
          uint64_t acc = 0;
          uint32_t dsel = 255;
          for (uint32_t dg = 0; dg < 256; ++dg) {
            if (sm.c_hist[dg] == 0) continue;
            if (acc + sm.w_hist[dg] >= rem) { dsel = dg; break; }
            acc += sm.w_hist[dg];
          }
          sm.prefix |= uint64_t(dsel) << shift;
          sm.need = rem - acc;
        }
        __syncthreads();
        rem = sm.need;
      }
      thresh = sm.prefix;
    }
    // compact victims (stamp <= tau) with warp ballots; order by stamp (bitonic)
    for (uint32_t base = 0; base < n_slots; base += kThreads) {
      const uint32_t s = base + tid;
      bool v = false;
      if (s < n_slots) {
        const uint32_t f = S.flags[s];
        v = (f & F_IN_LRU) && !(f & F_LOCKED) && S.mark[s] != epoch && S.last[s] <= thresh;
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, v);
      uint32_t wbase = 0;
      if (lane == 0 && bal) wbase = atomicAdd(&sm.n_vict, __popc(bal));
      wbase = __shfl_sync(0xffffffffu, wbase, 0);
      if (v) {
        const uint32_t k = wbase + __popc(bal & ((1u << lane) - 1));
        if (k < kMaxVictims) {
          sm.vkey[k] = S.last[s];
          sm.vslot[k] = s;
        }
      }
    }
    __syncthreads();
    const uint32_t nv = sm.n_vict;
    if (nv > kMaxVictims) {  // victims are only selected so far: undo the inserts and report
      if (tid == 0) rollback_inserts(a, r_slot, sm.old_slots, CTL_CAPACITY);
      return;
    }
    uint32_t np2 = 1;
    while (np2 < nv) np2 <<= 1;
    for (uint32_t k = nv + tid; k < np2; k += kThreads) { sm.vkey[k] = ~uint64_t(0); sm.vslot[k] = kEmpty; }
    __syncthreads();
    for (uint32_t size = 2; size <= np2; size <<= 1)
      for (uint32_t stride = size / 2; stride > 0; stride >>= 1) {
        for (uint32_t k = tid; k < np2; k += kThreads) {
          const uint32_t j = k ^ stride;
          if (j > k) {
            const bool up = (k & size) == 0;
            if ((sm.vkey[k] > sm.vkey[j]) == up) {
              const uint64_t tk = sm.vkey[k]; sm.vkey[k] = sm.vkey[j]; sm.vkey[j] = tk;
              const uint32_t ts = sm.vslot[k]; sm.vslot[k] = sm.vslot[j]; sm.vslot[j] = ts;
            }
          }
        }
        __syncthreads();
      }
    for (uint32_t k = tid; k < nv; k += kThreads) {
      const uint32_t v = sm.vslot[k];
      sm.vnp[k] = (S.flags[v] & F_HAS_PAGES) ? S.npages[v] : 0;
    }
  }
  __syncthreads();

  // ---- 5. the interleaved evict-push / allocate-pop sequence of ensure_free + page
  //         allocation (manager.cpp:55, :121-126), as stack positions (thread 0) ----
  if (tid == 0) {
    const uint32_t i_end = sm.i_end, nv = sm.n_vict;
    uint32_t top = uint32_t(free0), vi = 0, ids = 0, lo = uint32_t(free0), hi = uint32_t(free0), scr = 0;
    for (uint32_t i = 0; i < i_end; ++i) {
      const uint32_t c = r_grow[i] + r_scr[i];
      while (top < c && vi < nv) {
        sm.vpos[vi] = top;
        sm.vreq[vi] = i;
        top += sm.vnp[vi++];
      }
      hi = max(hi, top);
      top -= c;
      r_pop[i] = top;
      lo = min(lo, top);
      r_nv[i] = vi;
      r_ids[i] = ids;
      ids += c;
      scr += r_scr[i];
    }
    if (sm.fail == CTL_REJECT_VICTIMS)
      for (; vi < nv; ++vi) {  // ensure_free of the failing request evicts everyone, then throws
        sm.vpos[vi] = top;
        sm.vreq[vi] = i_end;
        top += sm.vnp[vi];
        hi = max(hi, top);
      }
    sm.min_pos = lo;
    sm.max_pos = hi;
    sm.final_top = top;
    sm.scratch_total = sm.fail == CTL_OK ? scr : 0;
    sm.n_ids = ids;
    sm.n_ev = vi;  // evictions
  }
  __syncthreads();
  const uint32_t i_end = sm.i_end, n_ev = sm.n_ev, n_ids = sm.n_ids;
  // value at stack position x as seen by request i's pops: the latest victim push
  // (victims are ordered in time) covering x among those evicted up to request i,
  // else the stack's content before the batch
  auto stack_at = [&](uint32_t x, uint32_t nvic) -> uint32_t {
    for (int k = int(nvic) - 1; k >= 0; --k)
      if (x >= sm.vpos[k] && x < sm.vpos[k] + sm.vnp[k]) return S.ptab[size_t(sm.vslot[k]) * a.max_pages + (x - sm.vpos[k])];
    return S.stack[x];
  };
  // pops of every allocating request, in parallel: grow pages (appended to the
  // user's page list) then scratch pages; pop e of request i reads r_pop[i] + c_i - 1 - e
  for (uint32_t i = warp; i < i_end; i += kThreads / 32) {
    const uint32_t g = r_grow[i], c = g + r_scr[i], s = r_slot[i];
    for (uint32_t e = lane; e < c; e += 32) {
      const uint32_t pg = stack_at(r_pop[i] + c - 1 - e, r_nv[i]);
      a.ids[r_ids[i] + e] = pg;
      if (e < g) S.ptab[size_t(s) * a.max_pages + r_havei[i] + e] = pg;
    }
  }
  // eviction records (state before the eviction)
  for (uint32_t k = tid; k < n_ev; k += kThreads) {
    const uint32_t v = sm.vslot[k];
    const uint64_t dl = S.dev[v], pl = S.pers[v];
    a.evict[k] = CtlEvict{v, 0, sm.vnp[k], 0, dl > pl ? dl - pl : 0};
  }
  __syncthreads();
  // stack after the batch: positions [min_pos, final_top) take their last push;
  // scratch pages are released on top in request order (manager.cpp:196)
  const uint32_t lo = sm.min_pos, ftop = sm.final_top;
  for (uint32_t x = lo + tid; x < ftop; x += kThreads) {
    uint32_t val = kEmpty;
    for (int k = int(n_ev) - 1; k >= 0; --k)
      if (x >= sm.vpos[k] && x < sm.vpos[k] + sm.vnp[k]) { val = S.ptab[size_t(sm.vslot[k]) * a.max_pages + (x - sm.vpos[k])]; break; }
    if (val != kEmpty) S.stack[x] = val;  // else unchanged since before the batch
  }
  __syncthreads();  // victim page lists are read above before they are cleared below
  const uint32_t fail = sm.fail;
  if (fail == CTL_OK) {
    for (uint32_t i = warp; i < a.n; i += kThreads / 32) {
      // scratch ids of request i go to ftop + (scratch released before it)
      uint32_t before = 0;
      for (uint32_t j = 0; j < i; ++j) before += r_scr[j];
      const uint32_t c = r_grow[i] + r_scr[i];
      for (uint32_t e = r_grow[i] + lane; e < c; e += 32) S.stack[ftop + before + (e - r_grow[i])] = a.ids[r_ids[i] + e];
    }
  }
  for (uint32_t k = tid; k < n_ev; k += kThreads) {
    const uint32_t v = sm.vslot[k];
    S.npages[v] = 0;
    S.flags[v] &= ~(F_HAS_PAGES | F_IN_LRU);
    S.dev[v] = 0;
  }
  __syncthreads();
  // ---- 6. touches (stamps in request order), page-list lengths, and on success the
  //         end-of-batch commit_onload / finish_append (final projections) ----
  if (tid == 0) {
    const uint32_t touch_end = fail == CTL_OK ? a.n : sm.fail_at + 1;
    const uint64_t stamp0 = G.stamp;
    for (uint32_t i = 0; i < touch_end && i < a.n; ++i) {
      const uint32_t s = r_slot[i];
      S.last[s] = stamp0 + i + 1;
      S.flags[s] |= F_KNOWN | F_IN_LRU;
      if (i < i_end) {
        S.npages[s] = r_havei[i] + r_grow[i];  // last allocating occurrence wins
        S.flags[s] |= F_HAS_PAGES;
        a.plans[i].stamp = stamp0 + i + 1;
        a.plans[i].grow_off = r_ids[i];
        a.plans[i].grow_n = r_grow[i];
        a.plans[i].scratch_off = r_ids[i] + r_grow[i];
        a.plans[i].scratch_n = r_scr[i];
      }
    }
    G.stamp = stamp0 + min(touch_end, a.n);
  }
  for (uint32_t i = tid; i < i_end; i += kThreads) {
    if (r_first[i] != i) continue;
    const uint32_t s = r_slot[i];
    if (fail == CTL_OK) {
      S.dev[s] = p_dev[i];
      if (p_total[i] > S.total[s]) S.total[s] = p_total[i];
    }
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t top = fail == CTL_OK ? ftop + sm.scratch_total : ftop;
    G.top = top;
    CtlHdr h{};
    h.fail = int32_t(fail);
    h.fail_at = int32_t(fail == CTL_OK ? a.n : sm.fail_at);
    h.n_evict = n_ev;
    h.n_ids = n_ids;
    h.free_top = top;
    h.n_slots = G.n_slots;
    h.stamp = G.stamp;
    *a.hdr = h;
  }
}

}  // namespace

int DevCtl::init(uint32_t device_pages, uint32_t page_size, uint32_t chunk_size, bool hier, uint32_t max_users,
                 uint32_t max_pages_per_user, uint64_t staging_tokens, std::string& err) {
  staging_tokens_ = staging_tokens;
  device_pages_ = device_pages;
  page_size_ = page_size;
  chunk_size_ = chunk_size;
  hier_ = hier;
  max_users_ = max_users;
  max_pages_ = max_pages_per_user;
  hash_cap_ = 1;
  while (hash_cap_ < 2 * max_users) hash_cap_ <<= 1;
  const size_t U = max_users;
  state_bytes_ = 256 + size_t(hash_cap_) * 8 + U * 8 * 4 + U * 4 * 4 + U * size_t(max_pages_) * 4 +
                 size_t(device_pages) * 4 + 16 * 64;
  if (cudaMalloc(&state_, state_bytes_) != cudaSuccess) { err = "device planner: table allocation failed"; return -1; }
  // globals, then the hash keys (all empty), then the free stack in the reference's
  // initial order (page 0 handed out first: stack[top-1] = 0)
  cudaMemset(state_, 0, state_bytes_);
  char* b = static_cast<char*>(state_);
  cudaMemset(b + 256, 0xFF, size_t(hash_cap_) * 4);
  std::vector<uint32_t> stk(device_pages);
  for (uint32_t i = 0; i < device_pages; ++i) stk[i] = device_pages - 1 - i;
  const size_t stack_off = state_bytes_ - size_t(device_pages) * 4 - 16 * 64;
  cudaMemcpy(b + stack_off, stk.data(), stk.size() * 4, cudaMemcpyHostToDevice);
  Globals g{device_pages, 0, 0, 0, 0};
  cudaMemcpy(b, &g, sizeof(g), cudaMemcpyHostToDevice);
  if (cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking) != cudaSuccess || cudaEventCreate(&ev0_) != cudaSuccess ||
      cudaEventCreate(&ev1_) != cudaSuccess) {
    err = "device planner: stream/event creation failed";
    return -1;
  }
  cudaFuncSetAttribute(ctl_prepare_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (cudaGetLastError() != cudaSuccess) { err = "device planner: init failed"; return -1; }
  return 0;
}

DevCtl::~DevCtl() {
  if (st_) cudaStreamSynchronize(st_);
  if (state_) cudaFree(state_);
  if (io_dev_) cudaFree(io_dev_);
  if (io_host_) cudaFreeHost(io_host_);
  if (ev0_) cudaEventDestroy(ev0_);
  if (ev1_) cudaEventDestroy(ev1_);
  if (st_) cudaStreamDestroy(st_);
}

static size_t al(size_t x) { return (x + 255) & ~size_t(255); }

int DevCtl::prepare(const CtlReq* reqs, uint32_t n, const std::vector<CtlUpd>& upd, std::string& err) {
  const size_t smem = sizeof(Smem) + size_t(n) * 4 * 3 + 8 + size_t(n) * 8 * 5 + size_t(n) * 4 * 5;
  if (smem > 200 * 1024) { err = "device planner: batch too large"; return -1; }
  // io layout: [reqs | upd | hdr | plans | evict (max_users) | ids (device_pages)]
  const size_t o_req = 0, o_upd = al(o_req + n * sizeof(CtlReq)), o_hdr = al(o_upd + upd.size() * sizeof(CtlUpd));
  const size_t o_plan = al(o_hdr + sizeof(CtlHdr)), o_ev = al(o_plan + n * sizeof(CtlPlan));
  const size_t o_ids = al(o_ev + size_t(max_users_) * sizeof(CtlEvict));
  const size_t bytes = al(o_ids + size_t(device_pages_) * 4);
  if (bytes > io_bytes_) {
    if (io_dev_) cudaFree(io_dev_);
    if (io_host_) cudaFreeHost(io_host_);
    io_bytes_ = bytes;
    if (cudaMalloc(&io_dev_, bytes) != cudaSuccess || cudaHostAlloc((void**)&io_host_, bytes, 0) != cudaSuccess) {
      err = "device planner: io allocation failed";
      return -1;
    }
  }
  std::memcpy(io_host_ + o_req, reqs, n * sizeof(CtlReq));
  if (!upd.empty()) std::memcpy(io_host_ + o_upd, upd.data(), upd.size() * sizeof(CtlUpd));
  char* d = static_cast<char*>(io_dev_);
  cudaMemcpyAsync(d, io_host_, o_hdr, cudaMemcpyHostToDevice, st_);
  // tables
  char* b = static_cast<char*>(state_);
  const size_t U = max_users_;
  Args a{};
  size_t off = 0;
  a.s.g = reinterpret_cast<Globals*>(b);
  off = 256;
  a.s.keys = reinterpret_cast<uint32_t*>(b + off); off += size_t(hash_cap_) * 4;
  a.s.vals = reinterpret_cast<uint32_t*>(b + off); off += size_t(hash_cap_) * 4;
  a.s.total = reinterpret_cast<uint64_t*>(b + off); off += U * 8;
  a.s.dev = reinterpret_cast<uint64_t*>(b + off); off += U * 8;
  a.s.pers = reinterpret_cast<uint64_t*>(b + off); off += U * 8;
  a.s.last = reinterpret_cast<uint64_t*>(b + off); off += U * 8;
  a.s.flags = reinterpret_cast<uint32_t*>(b + off); off += U * 4;
  a.s.npages = reinterpret_cast<uint32_t*>(b + off); off += U * 4;
  a.s.mark = reinterpret_cast<uint32_t*>(b + off); off += U * 4;
  a.s.firsti = reinterpret_cast<uint32_t*>(b + off); off += U * 4;
  a.s.ptab = reinterpret_cast<uint32_t*>(b + off); off += U * size_t(max_pages_) * 4;
  a.s.stack = reinterpret_cast<uint32_t*>(b + off);
  a.reqs = reinterpret_cast<const CtlReq*>(d + o_req);
  a.n = n;
  a.upd = reinterpret_cast<const CtlUpd*>(d + o_upd);
  a.n_upd = uint32_t(upd.size());
  a.hdr = reinterpret_cast<CtlHdr*>(d + o_hdr);
  a.plans = reinterpret_cast<CtlPlan*>(d + o_plan);
  a.evict = reinterpret_cast<CtlEvict*>(d + o_ev);
  a.ids = reinterpret_cast<uint32_t*>(d + o_ids);
  a.device_pages = device_pages_;
  a.page_size = page_size_;
  a.chunk_size = chunk_size_;
  a.max_users = max_users_;
  a.max_pages = max_pages_;
  a.hash_mask = hash_cap_ - 1;
  a.hier = hier_ ? 1 : 0;
  a.staging_tokens = staging_tokens_;
  cudaEventRecord(ev0_, st_);
  ctl_prepare_kernel<<<1, kThreads, smem, st_>>>(a);
  cudaEventRecord(ev1_, st_);
  // decisions back: header + plans + the first evictions / ids in one copy, the rest if needed
  const size_t ev_guess = std::min<size_t>(max_users_, 256), ids_guess = std::min<size_t>(device_pages_, 16384);
  cudaMemcpyAsync(io_host_ + o_hdr, d + o_hdr, o_ev - o_hdr + ev_guess * sizeof(CtlEvict), cudaMemcpyDeviceToHost, st_);
  cudaMemcpyAsync(io_host_ + o_ids, d + o_ids, ids_guess * 4, cudaMemcpyDeviceToHost, st_);
  if (cudaStreamSynchronize(st_) != cudaSuccess) {
    err = std::string("device planner: ") + cudaGetErrorString(cudaGetLastError());
    return -1;
  }
  std::memcpy(&hdr_, io_host_ + o_hdr, sizeof(CtlHdr));
  if (hdr_.n_evict > ev_guess)
    cudaMemcpy(io_host_ + o_ev, d + o_ev, size_t(hdr_.n_evict) * sizeof(CtlEvict), cudaMemcpyDeviceToHost);
  if (hdr_.n_ids > ids_guess) cudaMemcpy(io_host_ + o_ids, d + o_ids, size_t(hdr_.n_ids) * 4, cudaMemcpyDeviceToHost);
  plans_ = reinterpret_cast<CtlPlan*>(io_host_ + o_plan);
  evict_ = reinterpret_cast<CtlEvict*>(io_host_ + o_ev);
  ids_ = reinterpret_cast<uint32_t*>(io_host_ + o_ids);
  float ms = 0;
  cudaEventElapsedTime(&ms, ev0_, ev1_);
  last_ms_ = ms;
  if (hdr_.fail == CTL_CAPACITY) {  // rolled back on the device: the tables are as before the batch
    err = "device planner: capacity exceeded (max_users / max_user_pages / 4096 victims per batch)";
    return -1;
  }
  if (hdr_.fail == CTL_STAGING) {
    err = "onload buffer: batch exceeds staging capacity";
    return -1;
  }
  return 0;
}

}  // namespace mtkv_b200
