// Host-side planning of one batch's attention work (both attention kernels).
//
// tcgen05 path: every (request, head, 128-row query tile) segment needs the
// 128-key tiles of its visible logical key space (incremental attention of the
// fresh rows over the cached prefix + themselves, reference model.cpp:104).
// Per head, the concatenation of the segments' tiles is cut into contiguous,
// equal-length ranges, one per persistent CTA (sibling CTAs of the H heads run
// aligned ranges), so every SM streams the same number of K/V bytes regardless
// of how history lengths are distributed over the batch; a range that crosses a
// segment boundary becomes several pieces.
// Each piece yields one partial slot; the combine in gate_norm_kernel merges a
// segment's slots.
//
// mma.sync path (head_dim < 64): one CTA per (request, head, query tile, key
// split of split_keys positions), one slot per split.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "kernels.cuh"

namespace mtkv_b200 {

constexpr double kPieceCostDefault = 2.0;

void plan_attention(ReqDev* reqs, uint32_t n, const PoolGeom& g, bool tc, uint32_t ctas, AttnPlan& P, bool pair) {
  P.pair = tc && pair;
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
      R.qtiles = (R.n_q - R.q_skip + kTcBM - 1) / kTcBM;
      R.seg0 = uint32_t(P.segs.size());
      R.split_keys = 0;
      // logical key space: user keys [0, KA) padded to a page boundary, then candidates
      const uint64_t KA = R.start + R.n_hist, KAp = (KA + S - 1) / S * S;
      for (uint32_t h = 0; h < H; ++h)
        for (uint32_t qt = 0; qt < R.qtiles; ++qt) {
          const uint64_t q_end = std::min<uint64_t>(R.n_q, R.q_skip + uint64_t(qt + 1) * kTcBM);
          const uint64_t pos_last = R.start + q_end - 1;
          const uint64_t k_vis = pos_last >= KA ? KAp + (pos_last - KA + 1) : pos_last + 1;
          const uint32_t nt = uint32_t((k_vis + kTcBN - 1) / kTcBN);
          P.segs.push_back(AttnSeg{r, h, qt, nt, 0, 0});
          total += nt;
        }
    }
    if (total == 0) return;
    // Head siblings: the H heads of a (request, query tile) read the two (or H)
    // column blocks of the same pool rows. List k holds head k's segments in the
    // same (request, query tile) order, all lists have the same length, and CTA
    // c*H + k takes range c of list k, so the H sibling CTAs stream the same
    // DRAM rows at the same time (measured: 64.7 us vs 78.6 us per launch with
    // one flat list on the bench layer).
    // MTKV_ATTN_PART (measurement switch): heads (default) | flat | alt
    static const int part = [] {
      const char* e = std::getenv("MTKV_ATTN_PART");
      if (e && std::string(e) == "flat") return 1;
      if (e && std::string(e) == "alt") return 2;
      return 0;
    }();
    const uint32_t hg = part == 1 ? 1 : part == 2 ? 2 : (H >= 2 && H <= 8 && ctas >= 2 * H) ? H : 1;
    std::vector<std::vector<uint32_t>> lists(hg);
    std::vector<uint64_t> len(hg, 0);
    std::vector<std::vector<std::pair<uint32_t, uint32_t>>> spans(hg);  // (lo, hi) per listed segment
    // unit partner (paired kernel): B segment of each listed A segment, else kNoPart
    std::vector<std::vector<uint32_t>> partner(hg);
    if (part == 2 && !P.pair) {
      // alternate: segments in (request, head, query tile) order go to the
      // shorter of two lists, cut to even them out
      for (uint32_t sg = 0; sg < P.segs.size(); ++sg)
        for (uint32_t lo = 0, nt = P.segs[sg].n_tiles; lo < nt;) {
          const uint32_t k = len[0] <= len[1] ? 0 : 1;
          const uint64_t gap = len[1 - k] - len[k];
          const uint32_t take = uint32_t(gap ? std::min<uint64_t>(nt - lo, gap) : nt - lo);
          lists[k].push_back(sg);
          spans[k].push_back({lo, lo + take});
          len[k] += take;
          lo += take;
        }
      for (uint32_t k = 0; k < hg; ++k) partner[k].assign(lists[k].size(), kNoPart);
    } else {
      // pair: query tiles (2j, 2j+1) of a (request, head) form one unit over
      // the later tile's key tiles (the earlier one's are a prefix of them)
      for (uint32_t r = 0; r < n; ++r)
        for (uint32_t qt = 0; qt < reqs[r].qtiles; qt += P.pair ? 2 : 1)
          for (uint32_t h = 0; h < H; ++h) {
            const uint32_t sg = reqs[r].seg0 + h * reqs[r].qtiles + qt;
            const bool two = P.pair && qt + 1 < reqs[r].qtiles;
            const uint32_t nt = P.segs[two ? sg + 1 : sg].n_tiles;
            lists[h % hg].push_back(sg);
            partner[h % hg].push_back(two ? sg + 1 : kNoPart);
            spans[h % hg].push_back({0, nt});
            len[h % hg] += nt;
          }
    }
    const uint64_t G = std::max<uint64_t>(hg, std::min<uint64_t>(ctas, total));
    const uint32_t groups = uint32_t(G / hg);
    // Ranges are cut by cost, not tiles: a piece costs its tiles plus a fixed
    // overhead (its Q load, pipeline refill and O/lse epilogue: measured ~2.7 us
    // = ~2.2 tiles on a prefill, where a CTA's end time tracked its piece count
    // with r = 0.98 under tile-count cutting). MTKV_ATTN_PIECE_COST (in tiles;
    // 0 = tile-count cutting) is the A/B switch.
    static const double pe_cost = [] {
      const char* e = std::getenv("MTKV_ATTN_PIECE_COST");
      const double v = e ? std::atof(e) : kPieceCostDefault;
      return v >= 0.0 && v < 64.0 ? v : kPieceCostDefault;
    }();
    double max_cost = 0;
    for (uint32_t k = 0; k < hg; ++k) max_cost = std::max(max_cost, double(len[k]) + pe_cost * double(lists[k].size()));
    // every CTA boundary may split one segment (one more piece)
    const double quota = std::ceil((max_cost + pe_cost * groups) / groups);
    std::vector<std::vector<std::vector<AttnPiece>>> R(hg, std::vector<std::vector<AttnPiece>>(groups));
    for (uint32_t k = 0; k < hg; ++k) {
      uint32_t c = 0;
      double room = quota;
      for (size_t li = 0; li < lists[k].size(); ++li)
        for (uint32_t sg = lists[k][li], lo = spans[k][li].first, hi = spans[k][li].second; lo < hi;) {
          if (room < pe_cost + 1.0 && c + 1 < groups) { ++c; room = quota; }
          const uint32_t take = c + 1 == groups ? hi - lo
              : uint32_t(std::min<double>(hi - lo, std::max(1.0, std::floor(room - pe_cost))));
          AttnPiece pc{};
          pc.seg = sg;
          pc.lo = lo;
          pc.hi = lo + take;
          pc.part_b = partner[k][li];  // B's segment for now (its slot below)
          pc.na = P.segs[sg].n_tiles;
          R[k][c].push_back(pc);
          lo += take;
          room -= take + pe_cost;
        }
    }
    P.cta_off.push_back(0);
    for (uint32_t c = 0; c < groups; ++c)
      for (uint32_t k = 0; k < hg; ++k) {
        for (const AttnPiece& pc : R[k][c]) P.pieces.push_back(pc);
        P.cta_off.push_back(uint32_t(P.pieces.size()));
      }
    // slots: a segment's pieces may sit in different CTAs' lists; give every
    // segment a contiguous slot range
    std::vector<uint32_t> npc(P.segs.size(), 0);
    for (const AttnPiece& pc : P.pieces) {
      if (pc.lo < pc.na) ++npc[pc.seg];  // the A tile has key tiles in this piece
      if (pc.part_b != kNoPart) ++npc[pc.part_b];
    }
    for (uint32_t sg = 0; sg < P.segs.size(); ++sg) {
      P.segs[sg].part_base = P.n_slots;
      P.segs[sg].n_parts = npc[sg];
      P.n_slots += npc[sg];
    }
    std::vector<uint32_t> used(P.segs.size(), 0);
    for (AttnPiece& pc : P.pieces) {
      pc.part = pc.lo < pc.na ? P.segs[pc.seg].part_base + used[pc.seg]++ : kNoPart;
      if (pc.part_b != kNoPart) pc.part_b = P.segs[pc.part_b].part_base + used[pc.part_b]++;
      const AttnSeg& sg = P.segs[pc.seg];
      const ReqDev& R = reqs[sg.req];
      pc.head = sg.head;
      pc.qtile = sg.qtile;
      pc.q_row0 = R.q_row0;
      pc.n_q = R.n_q;
      pc.n_hist = R.n_hist;
      pc.n_cand = R.n_cand;
      pc.pages_off = R.pages_off;
      pc.scratch_off = R.scratch_off;
      pc.n_scratch = R.n_scratch;
      pc.q_skip = R.q_skip;
      pc.start = R.start;
      pc.dep_start = R.dep_start;
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

// ---- C-ABI self-check of the planner (host only; used by the CPU tests) ----
#include "../../include/mtkv_b200.h"

extern "C" int mtkv_attention_plan_check(uint32_t n, const uint32_t* n_hist, const uint32_t* n_cand,
                                         const uint64_t* start, uint32_t H, uint32_t D, uint32_t S, uint32_t ctas,
                                         int tc, uint32_t* out_stats) {
  using namespace mtkv_b200;
  PoolGeom g{};
  g.H = H;
  g.D = D;
  g.d = H * D;
  g.S = S;
  g.L = 1;
  std::vector<ReqDev> rq(n);
  uint32_t rows = 0;
  for (uint32_t r = 0; r < n; ++r) {
    rq[r] = ReqDev{};
    rq[r].q_row0 = rows;
    rq[r].n_hist = n_hist[r];
    rq[r].n_cand = n_cand[r];
    rq[r].n_q = n_hist[r] + n_cand[r];
    rq[r].start = start[r];
    rows += rq[r].n_q;
  }
  AttnPlan P;
  plan_attention(rq.data(), n, g, tc != 0, ctas, P, tc == 2);  // tc = 2: paired query tiles
  // every segment: its slots are contiguous and its tiles are covered exactly once
  std::vector<std::vector<uint32_t>> cover(P.segs.size());
  for (size_t s = 0; s < P.segs.size(); ++s) cover[s].assign(tc ? P.segs[s].n_tiles : 1, 0);
  uint64_t tiles = 0, max_cta = 0;
  if (tc) {
    if (P.cta_off.empty() || P.cta_off.front() != 0 || P.cta_off.back() != P.pieces.size()) return 1;
    for (size_t c = 0; c + 1 < P.cta_off.size(); ++c) {
      uint64_t t = 0;
      for (uint32_t i = P.cta_off[c]; i < P.cta_off[c + 1]; ++i) {
        const AttnPiece& pc = P.pieces[i];
        if (pc.seg >= P.segs.size() || pc.lo >= pc.hi) return 2;
        const AttnSeg& sg = P.segs[pc.seg];
        const uint32_t ha = std::min(pc.hi, pc.na);
        if (pc.lo < ha && (pc.part < sg.part_base || pc.part + 1 > sg.part_base + sg.n_parts)) return 3;
        if (pc.lo >= ha && pc.part != kNoPart) return 3;
        for (uint32_t x = pc.lo; x < ha; ++x) ++cover[pc.seg][x];
        if (pc.part_b != kNoPart) {  // paired: B = the next query tile of the same (request, head)
          const uint32_t sb = pc.seg + 1;
          if (!P.pair || sb >= P.segs.size() || P.segs[sb].req != sg.req || P.segs[sb].head != sg.head ||
              P.segs[sb].qtile != sg.qtile + 1 || pc.hi > P.segs[sb].n_tiles)
            return 8;
          if (pc.part_b < P.segs[sb].part_base || pc.part_b + 1 > P.segs[sb].part_base + P.segs[sb].n_parts) return 3;
          for (uint32_t x = pc.lo; x < pc.hi; ++x) ++cover[sb][x];
        } else if (pc.hi > sg.n_tiles) {
          return 2;
        }
        t += pc.hi - pc.lo;
      }
      tiles += t;
      max_cta = std::max(max_cta, t);
    }
    for (auto& cv : cover)
      for (uint32_t c : cv)
        if (c != 1) return 4;
  } else {
    for (const AttnItem& it : P.items) {
      const ReqDev& R = rq[it.req];
      const uint32_t sg = R.seg0 + it.head * R.qtiles + it.qtile;
      if (sg >= P.segs.size() || it.split >= P.segs[sg].n_parts) return 5;
    }
  }
  uint32_t slots = 0;
  for (const AttnSeg& sg : P.segs) {
    if (sg.part_base != slots) return 6;  // contiguous, in segment order
    slots += sg.n_parts;
  }
  if (slots != P.n_slots) return 7;
  if (out_stats) {
    out_stats[0] = uint32_t(P.segs.size());
    out_stats[1] = uint32_t(tc ? P.pieces.size() : P.items.size());
    out_stats[2] = uint32_t(tiles);
    out_stats[3] = uint32_t(max_cta);
    out_stats[4] = P.n_ctas();
  }
  return 0;
}
