// Host-side planning of one batch's attention work (both attention kernels).
//
// tcgen05 path: every (request, head, 128-row query tile) segment needs the
// 64-key tiles of its visible logical key space (incremental attention of the
// fresh rows over the cached prefix + themselves, reference model.cpp:104).
// The concatenation of all segments' tiles is cut into `ctas` contiguous,
// equal-length ranges, one per persistent CTA, so every SM streams the same
// number of K/V bytes regardless of how history lengths are distributed over
// the batch; a range that crosses a segment boundary becomes several pieces.
// Each piece yields two partial slots (one per softmax pipeline); the combine
// in gate_norm_kernel merges a segment's slots.
//
// mma.sync path (head_dim < 64): one CTA per (request, head, query tile, key
// split of split_keys positions), one slot per split.
#include <algorithm>

#include "kernels.cuh"

namespace mtkv_b200 {

void plan_attention(ReqDev* reqs, uint32_t n, const PoolGeom& g, bool tc, uint32_t ctas, AttnPlan& P) {
  P.segs.clear();
  P.pieces.clear();
  P.cta_off.clear();
  P.items.clear();
  P.n_slots = 0;
  const uint32_t S = g.S, H = g.H;
  if (tc) {
    P.bm = kTcBM;
    uint64_t total = 0;
    for (uint32_t r = 0; r < n; ++r) {
      ReqDev& R = reqs[r];
      R.qtiles = (R.n_q + kTcBM - 1) / kTcBM;
      R.seg0 = uint32_t(P.segs.size());
      R.split_keys = 0;
      // logical key space: user keys [0, KA) padded to a page boundary, then candidates
      const uint64_t KA = R.start + R.n_hist, KAp = (KA + S - 1) / S * S;
      for (uint32_t h = 0; h < H; ++h)
        for (uint32_t qt = 0; qt < R.qtiles; ++qt) {
          const uint64_t q_end = std::min<uint64_t>(R.n_q, uint64_t(qt + 1) * kTcBM);
          const uint64_t pos_last = R.start + q_end - 1;
          const uint64_t k_vis = pos_last >= KA ? KAp + (pos_last - KA + 1) : pos_last + 1;
          const uint32_t nt = uint32_t((k_vis + kTcBN - 1) / kTcBN);
          P.segs.push_back(AttnSeg{r, h, qt, nt, 0, 0});
          total += nt;
        }
    }
    if (total == 0) return;
    const uint64_t G = std::max<uint64_t>(1, std::min<uint64_t>(ctas, total));
    const uint64_t quota = (total + G - 1) / G;
    P.cta_off.push_back(0);
    uint64_t room = quota;
    for (uint32_t s = 0; s < P.segs.size(); ++s) {
      const uint32_t nt = P.segs[s].n_tiles;
      for (uint32_t lo = 0; lo < nt;) {
        const uint32_t take = uint32_t(std::min<uint64_t>(nt - lo, room));
        P.pieces.push_back(AttnPiece{s, lo, lo + take, 0});
        lo += take;
        room -= take;
        if (room == 0) {
          P.cta_off.push_back(uint32_t(P.pieces.size()));
          room = quota;
        }
      }
    }
    if (P.cta_off.back() != P.pieces.size()) P.cta_off.push_back(uint32_t(P.pieces.size()));
    for (AttnPiece& pc : P.pieces) {  // a segment's pieces are consecutive -> contiguous slots
      AttnSeg& sg = P.segs[pc.seg];
      if (sg.n_parts == 0) sg.part_base = P.n_slots;
      pc.part = P.n_slots;
      P.n_slots += 2;
      sg.n_parts += 2;
    }
    return;
  }
  // mma.sync path: 64/128-row query tiles over positions, 512-key splits for
  // short query sets (one tile per request streams the prefix once)
  uint32_t max_q = 0;
  for (uint32_t r = 0; r < n; ++r) max_q = std::max(max_q, reqs[r].n_q);
  P.bm = max_q > 64 ? 128 : 64;
  for (uint32_t r = 0; r < n; ++r) {
    ReqDev& R = reqs[r];
    const uint64_t T = R.start + R.n_q;
    R.split_keys = R.n_q <= 256 ? 512u : uint32_t(std::min<uint64_t>(T + 128, 0xFFFFFF00ull));
    const uint32_t splits = uint32_t((T + R.split_keys - 1) / R.split_keys);
    R.qtiles = (R.n_q + P.bm - 1) / P.bm;
    R.seg0 = uint32_t(P.segs.size());
    for (uint32_t h = 0; h < H; ++h)
      for (uint32_t qt = 0; qt < R.qtiles; ++qt) {
        P.segs.push_back(AttnSeg{r, h, qt, 0, P.n_slots, splits});
        P.n_slots += splits;
        for (uint32_t sp = 0; sp < splits; ++sp) P.items.push_back(AttnItem{r, h, qt, sp});
      }
  }
}

}  // namespace mtkv_b200
