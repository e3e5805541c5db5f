// Paired-query-tile attention for prefill-shaped work (sm_100a, head_dim 128).
//
// The re-encoded head of a split host hit, a recomputed miss and a prefill are
// causal self-attention over thousands of rows: per (query tile, key tile) the
// work is two 128x128x128 MMAs plus 16 384 exponentials, and the one-tile
// kernel (attn_tc.cu) is softmax-bound there (its two softmax warpgroups split
// the columns of one S tile and meet at a row-max barrier every tile, so the
// MUFU pipe idles while both load S and exchange maxima).
// This kernel pairs the query tiles 2j and 2j+1 of one (request, head): they
// share every K/V tile (each tile loaded once for 256 rows), and each has its
// own softmax warpgroup that owns whole rows (thread = row, all 128 columns:
// no exchange), so while warpgroup A exponentiates its tile the tensor core
// runs B's S / PV MMAs and vice versa (the ping-pong of FlashAttention-4).
// A request with one query tile (or the odd last tile) is a piece without B.
// Measured variant, selected by MTKV_ATTN_PAIR=1 (default: the one-tile kernel,
// which it does not beat: 254 vs 248 us on a 24 x 4K prefill, 103 vs 78 us on
// the decode layer).
//
// Persistent, one CTA per SM, 384 threads:
//   warp 0      K/V producer: page-granular TMA out of the paged pool into one
//               ring of K(t), V(t), K(t+1), ... stages (released in that order)
//   warp 1      MMA issuer: S_X = Q_X K^T (both operands in shared memory),
//               O_X += P_X V (P in TMEM over S_X), order per tile t:
//               PV_A(t) S_A(t+1) PV_B(t) S_B(t+1)
//   warp 2      TMEM allocator, then Q loader (both query tiles of a piece)
//   warps 4..7  softmax of query tile A (thread r = row r = TMEM lane r)
//   warps 8..11 softmax of query tile B
// TMEM: S_A | S_B | O_A | O_B (4 x 128 fp32 columns).
// Row sums are accumulated in registers (each thread owns its row).
// Plan: attn_plan.cpp (pair = true): pieces carry part (tile A's slot), part_b
// (tile B's slot or kNoPart) and na (A's visible key tiles: A is active for
// tiles t < na of the piece, B for all of them).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>

#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace mtkv_b200 {

using namespace tc;

namespace pair {
constexpr int BM = 128, BN = 128, D = 128;
constexpr uint32_t KBLK = BN * 128;         // 128 rows x 128 B (64 bf16)
constexpr uint32_t T_BYTES = 2 * KBLK;      // one K, V or Q tile (D = 128: two 64-column blocks)
constexpr int NS = 5;                       // K/V ring stages
constexpr uint32_t S_COL = 0, O_COL = 2 * BN;
constexpr size_t SMEM = size_t(2 + NS) * T_BYTES + 256;
static_assert(SMEM <= 232448, "shared memory budget");
}  // namespace pair

#define PAIR_TR(kind, t)                                                                  \
  do {                                                                                    \
    if (TR && blockIdx.x < kTraceCtas && (t) < kTraceTiles)                               \
      a.trace[((size_t)blockIdx.x * kTraceKinds + (kind)) * kTraceTiles + (t)] = gtime(); \
  } while (0)

// TR: per-CTA event trace (MTKV_ATTN_TRACE; kinds as attn_tc.cu for query tile A:
// 0 K issued, 1 S_A issued, 2 PV_A issued, 3 S_A ready, 6 row max, 7 P stored,
// 8 O rescaled, 4 P_A arrived, 9 S_A wait entered, 10 p_full_A wait entered,
// 11 S_B ready; 5: 0 start, 1 init done, 2 end)
template <bool TR>
__global__ void __launch_bounds__(384, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap pool_map, const __grid_constant__ CUtensorMap q_map,
                     AttnArgs a) {
  using namespace pair;
  constexpr float kRescale = 8.f;  // lazy rescale threshold (log2 units)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sQ = smem_raw;                 // [2] query tiles (A, B)
  uint8_t* sR = sQ + 2 * T_BYTES;         // [NS] K/V ring
  uint64_t* bars = reinterpret_cast<uint64_t*>(sR + NS * T_BYTES);
  uint64_t* full = bars;                  // [NS]
  uint64_t* empty = full + NS;            // [NS]
  uint64_t* q_full = empty + NS;
  uint64_t* q_empty = q_full + 1;
  uint64_t* s_full = q_empty + 1;         // [2] S_X computed
  uint64_t* p_full = s_full + 2;          // [2] P_X in TMEM (+ O_X rescaled): 4 warps
  uint64_t* o_done = p_full + 2;          // [2] PV_X completed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const PoolGeom& g = a.g;
  const uint32_t S = g.S;
  const uint32_t pb = a.cta_off[blockIdx.x], pe = a.cta_off[blockIdx.x + 1];
  if (threadIdx.x == 0) PAIR_TR(5, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int x = 0; x < 2; ++x) {
      mbar_init(&s_full[x], 1);
      mbar_init(&p_full[x], 4);
      mbar_init(&o_done[x], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tmem_slot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) PAIR_TR(5, 1);
  if (a.trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    // ---------------- K/V producer: ring positions K(0) V(0) K(1) V(1) ... ----------------
    const uint32_t ppt = BN / S;
    uint32_t gp = 0, st = 0, ph = 0;
    bool dep_done = false;
    auto acquire = [&]() -> uint8_t* {
      if (lane == 0) {
        if (gp >= uint32_t(NS)) mbar_wait(&empty[st], ph ^ 1);
        mbar_expect_tx(&full[st], T_BYTES);
      }
      __syncwarp();
      return sR + st * T_BYTES;
    };
    auto advance = [&]() {
      ++gp;
      if (++st == uint32_t(NS)) { st = 0; ph ^= 1; }
    };
    // pool row of a logical page of piece P (K plane; V = + S), or an
    // out-of-bounds row (TMA zero fill)
    auto row_of = [&](const AttnPiece& P, uint64_t lp) -> int {
      const uint32_t user_pages = uint32_t((P.start + P.n_hist + S - 1) / S);
      uint32_t page;
      if (lp < user_pages) page = a.pages[P.pages_off + uint32_t(lp)];
      else if (lp - user_pages < P.n_scratch && (lp - user_pages) * S < P.n_cand)
        page = a.pages[P.scratch_off + uint32_t(lp - user_pages)];
      else return -int(S) * 4;
      return int(((uint64_t(a.layer) * g.num_pages + page) * 2) * S);
    };
    // L2 prefetch cursor kPF tiles ahead of the loads (crossing piece
    // boundaries): a tile's TMA loads then hit L2 instead of waiting ~5-10 us
    // on DRAM behind a ring that covers only ~2.5 tiles
    constexpr uint32_t kPF = 4;
    uint32_t f_pc = pb, f_t = 0, f_t0 = 0, f_done = 0;
    int f_rows = 0;
    AttnPiece F{};
    auto f_load = [&]() {
      if (f_pc < pe) {
        F = a.pieces[f_pc];
        f_t = f_t0 = F.lo;
        f_rows = row_of(F, uint64_t(F.lo) * ppt + lane);
      }
    };
    f_load();
    auto prefetch_to = [&](uint32_t target) {  // issue prefetches for CTA tiles [f_done, target)
      while (f_done < target && f_pc < pe) {
        if (!dep_done && uint64_t(f_t + 1) * BN > F.dep_start) return;  // not before this layer's appends
        if ((f_t - f_t0) * ppt >= 32) {
          f_t0 = f_t;
          f_rows = row_of(F, uint64_t(f_t) * ppt + lane);
        }
        const int row = __shfl_sync(0xffffffffu, f_rows, ((f_t - f_t0) * ppt + lane) & 31);
        if (lane < ppt && row >= 0) {
          const int c = int(F.head * D);
          tma_prefetch_2d(&pool_map, c, row);
          tma_prefetch_2d(&pool_map, c + 64, row);
          tma_prefetch_2d(&pool_map, c, row + int(S));
          tma_prefetch_2d(&pool_map, c + 64, row + int(S));
        }
        ++f_done;
        if (++f_t == F.hi) {
          ++f_pc;
          f_load();
        }
      }
    };
    uint32_t g_t = 0;  // CTA tile index of the loads
    for (uint32_t pc = pb; pc < pe; ++pc) {
      const AttnPiece P = a.pieces[pc];
      const uint32_t col = P.head * D;
      uint32_t cache_t0 = P.lo;
      int rows_cache = row_of(P, uint64_t(P.lo) * ppt + lane);
      for (uint32_t t = P.lo; t < P.hi; ++t, ++g_t) {
        if ((t - cache_t0) * ppt >= 32) {
          cache_t0 = t;
          rows_cache = row_of(P, uint64_t(t) * ppt + lane);
        }
        if (!dep_done && uint64_t(t + 1) * BN > P.dep_start) {  // tile holds keys this layer's GEMM appends
          asm volatile("griddepcontrol.wait;" ::: "memory");
          dep_done = true;
        }
        prefetch_to(g_t + 1 + kPF);
        if (lane == 0) PAIR_TR(0, gp / 2);
#pragma unroll 1
        for (int kv = 0; kv < 2; ++kv) {
          uint8_t* dst = acquire();
          for (uint32_t i = 0; i < ppt; ++i) {
            int row = __shfl_sync(0xffffffffu, rows_cache, (t - cache_t0) * ppt + i);
            if (kv && row >= 0) row += int(S);
            if (lane == 0) {
              tma_load_2d(dst + i * S * 128, &pool_map, int(col), row, &full[st]);
              tma_load_2d(dst + KBLK + i * S * 128, &pool_map, int(col + 64), row, &full[st]);
            }
          }
          advance();
        }
      }
    }
  } else if (warp == 2) {
    // ---------------- Q loader: both query tiles of each piece ----------------
    asm volatile("griddepcontrol.wait;" ::: "memory");  // Q is written by the projection GEMM
    if (lane == 0) {
      uint32_t n = 0;
      for (uint32_t pc = pb; pc < pe; ++pc, ++n) {
        const AttnPiece P = a.pieces[pc];
        const bool has_b = P.part_b != kNoPart;
        if (n) mbar_wait(q_empty, (n - 1) & 1);  // every S MMA of the previous piece completed
        mbar_expect_tx(q_full, (has_b ? 2 : 1) * T_BYTES);
        const int row = int(P.q_row0 + P.q_skip + P.qtile * BM);
        const int col = int(P.head * D);
        tma_load_2d(sQ, &q_map, col, row, q_full);
        tma_load_2d(sQ + KBLK, &q_map, col + 64, row, q_full);
        if (has_b) {
          tma_load_2d(sQ + T_BYTES, &q_map, col, row + BM, q_full);
          tma_load_2d(sQ + T_BYTES + KBLK, &q_map, col + 64, row + BM, q_full);
        }
        if (pc + 1 < pe) {  // the next piece's Q into L2 while this piece runs
          const AttnPiece Pn = a.pieces[pc + 1];
          const int rn = int(Pn.q_row0 + Pn.q_skip + Pn.qtile * BM), cn = int(Pn.head * D);
          tma_prefetch_2d(&q_map, cn, rn);
          tma_prefetch_2d(&q_map, cn + 64, rn);
          if (Pn.part_b != kNoPart) {
            tma_prefetch_2d(&q_map, cn, rn + BM);
            tma_prefetch_2d(&q_map, cn + 64, rn + BM);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // per tile c (K at ring position pos, V at pos + 1), next tile n:
    //   PV_A(c)  [S_A(n)]  PV_B(c)  release V(c)  [new piece: wait Q]  (S_A(n))  S_B(n)  release K(n)
    // S_X(n) overwrites S_X's buffer behind PV_X(c), which has read P_X(c) from
    // it (in-order tensor pipe); A's next S goes ahead of B's PV so warpgroup A
    // never waits for B's softmax.
    if (pe > pb) {
      constexpr uint32_t idesc_s =
          (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
      constexpr uint32_t idesc_o =
          (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(D >> 3) << 17) | (uint32_t(BM >> 4) << 24);
      const bool leader = elect_one();
      const uint64_t dq0 = sdesc(s32(sQ), 16, 1024);
      const uint64_t dk0 = sdesc(s32(sR), 16, 1024), dv0 = sdesc(s32(sR), KBLK, 1024);
      struct Cur {
        uint32_t pc, t, hi, na;
        bool b;
      };
      auto load_cur = [&](uint32_t pc) -> Cur {
        Cur c{pc, 0, 0, 0, false};
        if (pc < pe) {
          const AttnPiece& P = a.pieces[pc];
          c.t = P.lo;
          c.hi = P.hi;
          c.na = P.na;
          c.b = P.part_b != kNoPart;
        }
        return c;
      };
      auto wait_stage = [&](uint32_t p) {
        mbar_wait(&full[p % NS], (p / NS) & 1);
        tc_after();
      };
      uint32_t ns_a = 0;
      auto issue_s = [&](uint32_t x, uint32_t kpos) {
        if (x == 0) PAIR_TR(9, ns_a);
        wait_stage(kpos);
        const uint64_t bk = dk0 + (((kpos % NS) * T_BYTES) >> 4);
        const uint64_t aq = dq0 + ((x * T_BYTES) >> 4);
        const uint32_t d_tmem = tmem + S_COL + x * BN;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = ((kk / 4) * KBLK + (kk % 4) * 32) >> 4;
          mma_f16_if(leader, d_tmem, aq + off, bk + off, idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit_if(leader, &s_full[x]);
        if (x == 0) { if (leader) PAIR_TR(1, ns_a); ++ns_a; }
      };
      uint32_t pf[2] = {0, 0};  // p_full waits per query tile
      bool first[2] = {true, true};  // next PV_X is the piece's first (overwrite O_X)
      auto issue_pv = [&](uint32_t x, uint32_t vpos) {
        if (x == 0) PAIR_TR(10, pf[0]);
        mbar_wait(&p_full[x], pf[x] & 1);
        ++pf[x];
        wait_stage(vpos);
        const uint64_t bv = dv0 + (((vpos % NS) * T_BYTES) >> 4);
        const uint32_t a_tmem = tmem + S_COL + x * BN;
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          mma_ts_if(leader, tmem + O_COL + x * D, a_tmem + kk * 8, bv + ((kk * 2048) >> 4), idesc_o,
                    (!first[x] || kk > 0) ? 1u : 0u);
        first[x] = false;
        mma_commit_if(leader, &o_done[x]);
        if (x == 0 && leader) PAIR_TR(2, pf[0] - 1);
      };
      uint32_t q_ph = 0, pos = 0;
      Cur c = load_cur(pb);
      mbar_wait(q_full, q_ph);
      q_ph ^= 1;
      tc_after();
      if (c.t < c.na) issue_s(0, pos);
      if (c.b) issue_s(1, pos);
      mma_commit_if(leader, &empty[pos % NS]);
      if (c.t + 1 == c.hi) mma_commit_if(leader, q_empty);
      for (;;) {
        Cur n = c;
        ++n.t;
        const bool boundary = n.t >= c.hi;
        if (boundary) n = load_cur(c.pc + 1);
        const bool more = n.pc < pe;
        const bool na = more && n.t < n.na, nb = more && n.b;
        const uint32_t npos = pos + 2;
        if (c.t < c.na) issue_pv(0, pos + 1);
        if (!boundary && na) issue_s(0, npos);
        if (c.b) issue_pv(1, pos + 1);
        mma_commit_if(leader, &empty[(pos + 1) % NS]);  // V(c) read by every PV of the tile
        if (!more) break;
        if (boundary) {
          first[0] = first[1] = true;
          mbar_wait(q_full, q_ph);  // the next piece's Q (its loader waited for q_empty)
          q_ph ^= 1;
          tc_after();
          if (na) issue_s(0, npos);
        }
        if (nb) issue_s(1, npos);
        mma_commit_if(leader, &empty[npos % NS]);  // K(n) read by every S of the tile
        if (n.t + 1 == n.hi) mma_commit_if(leader, q_empty);
        c = n;
        pos = npos;
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax: warpgroup x owns query tile x of each piece, thread = row ----------------
    const uint32_t x = (warp - 4) / 4;
    const uint32_t r = threadIdx.x % 128;
    const uint32_t lane_base = (32u * (warp % 4)) << 16;
    const uint32_t s_addr = tmem + lane_base + S_COL + x * BN;
    const uint32_t o_addr = tmem + lane_base + O_COL + x * D;
    uint32_t k = 0;  // tiles processed by this warpgroup (s_full / o_done phases)
    for (uint32_t pc = pb; pc < pe; ++pc) {
      const AttnPiece P = a.pieces[pc];
      if (x == 1 && P.part_b == kNoPart) continue;
      const uint32_t t_end = x == 0 ? min(P.hi, P.na) : P.hi;
      if (P.lo >= t_end) continue;
      const uint32_t part = x == 0 ? P.part : P.part_b;
      const uint64_t KA = P.start + P.n_hist;
      const uint64_t KAp = (KA + S - 1) / S * S;
      const uint32_t q0 = P.q_skip + (P.qtile + x) * BM;
      const uint32_t q_end = min(P.n_q, q0 + BM);
      const uint64_t pos_last = P.start + q_end - 1;
      const uint64_t k_vis = pos_last >= KA ? KAp + (pos_last - KA + 1) : pos_last + 1;
      const uint64_t k_hi = min(k_vis, uint64_t(t_end) * BN);
      const uint64_t pos_r = P.start + q0 + r;
      const uint64_t u_end = min(min(KA, k_hi), pos_r + 1);
      const uint64_t c_end = pos_r >= KA ? min(min(KAp + P.n_cand, KAp + (pos_r - KA + 1)), k_hi) : KAp;
      const uint64_t kb0 = uint64_t(P.lo) * BN;
      const int64_t span = int64_t(t_end - P.lo) * BN;
      auto rel = [&](uint64_t v) { return int(min(max(int64_t(v) - int64_t(kb0), int64_t(-1)), span)); };
      const int ue = rel(u_end), cl = rel(KAp), ce = rel(c_end);
      float m_ref = -INFINITY, l_run = 0.f;
      for (uint32_t t = P.lo; t < t_end; ++t, ++k) {
        mbar_wait(&s_full[x], k & 1);
        tc_after();
        const bool tr0 = threadIdx.x == 128, tr1 = threadIdx.x == 256;
        if (tr0) PAIR_TR(3, k);
        if (tr1) PAIR_TR(11, k);
        // pass 1: row max (64 columns per load); pass 2: exponentials per
        // 32-column chunk, the next chunk's load in flight (no 128-float row
        // held in registers: the softmax thread stays within 168 registers)
        const int kb = int(t - P.lo) * BN;
        const int cu = min(max(ue - kb, 0), BN), c_lo = min(max(cl - kb, 0), BN), c_hi = min(max(ce - kb, 0), BN);
        const bool full_tile = cu == BN;
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float v[64];
          tmem_ld32(s_addr + hh * 64, v);
          tmem_ld32(s_addr + hh * 64 + 32, v + 32);
          tmem_wait_ld();
          if (!full_tile) {
            // valid columns as a bit mask per 32-column chunk: one shift + select per
            // element (a per-element || compiled to a divergent branch each)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int c0 = hh * 64 + q * 32;
              const uint32_t bits = range_bits(-c0, cu - c0) | range_bits(c_lo - c0, c_hi - c0);
#pragma unroll
              for (int c = 0; c < 32; ++c) v[q * 32 + c] = (bits >> c) & 1u ? v[q * 32 + c] : -INFINITY;
            }
          }
#pragma unroll
          for (int c = 0; c < 64; ++c) m4[c & 3] = fmaxf(m4[c & 3], v[c]);
        }
        const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * a.scale_log2;
        float alpha = 1.f;
        if (mx > m_ref + kRescale) {
          alpha = m_ref == -INFINITY ? 0.f : ex2(m_ref - mx);
          m_ref = mx;
        }
        const float nmref = m_ref == -INFINITY ? 0.f : -m_ref;
        if (tr0) PAIR_TR(6, k);
        float l4[4] = {0.f, 0.f, 0.f, 0.f};
        float v0[32], v1[32];
        tmem_ld32(s_addr, v0);
        tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < BN / 32; ++h) {
          if (h + 1 < BN / 32) tmem_ld32(s_addr + (h + 1) * 32, (h & 1) ? v0 : v1);
          float* w = (h & 1) ? v1 : v0;
          if (!full_tile) {
            const int c0 = h * 32;
            const uint32_t bits = range_bits(-c0, cu - c0) | range_bits(c_lo - c0, c_hi - c0);
#pragma unroll
            for (int c = 0; c < 32; ++c) w[c] = (bits >> c) & 1u ? w[c] : -INFINITY;
          }
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const float p0 = ex2(fmaf(w[2 * c], a.scale_log2, nmref));
            const float p1 = ex2(fmaf(w[2 * c + 1], a.scale_log2, nmref));
            l4[(2 * c) & 3] += p0;
            l4[(2 * c + 1) & 3] += p1;
            pk[c] = pack2(p0, p1);
          }
          // P (bf16x2) over S columns [16h, 16h + 16): chunk h + 1's S columns
          // [32h + 32, ...) are not overwritten, and its load was issued first
          tmem_st16(s_addr + h * 16, pk);
          if (h + 1 < BN / 32) tmem_wait_ld();
        }
        if (tr0) PAIR_TR(7, k);
        l_run = l_run * alpha + ((l4[0] + l4[1]) + (l4[2] + l4[3]));
        if (t != P.lo) {  // PV_X(previous tile) must finish before O_X is rescaled
          mbar_wait(&o_done[x], (k - 1) & 1);
          tc_after();
          if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
              float o[32];
              tmem_ld32(o_addr + c * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] *= alpha;
              tmem_st32(o_addr + c * 32, o);
            }
          }
        }
        if (tr0) PAIR_TR(8, k);
        tmem_wait_st();
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[x]);
        if (tr0) PAIR_TR(4, k);
      }
      // ---- epilogue: O_X / l and lse (base 2) into slot `part` ----
      mbar_wait(&o_done[x], (k - 1) & 1);
      tc_after();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      const uint32_t qi = q0 + r;
      const bool valid = qi < q_end;
      float* dst = a.part_o + part_index(part, BM, r, 0, D);
      constexpr size_t chunk_stride = size_t(BM) * 4;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        tmem_ld32(o_addr + c * 32, o);
        tmem_wait_ld();
        if (valid) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(dst + (c * 8 + j) * chunk_stride) =
                make_float4(o[4 * j] * inv, o[4 * j + 1] * inv, o[4 * j + 2] * inv, o[4 * j + 3] * inv);
        }
      }
      if (valid) a.part_lse[size_t(part) * BM + r] = l_run > 0.f ? m_ref + log2f(l_run) : -INFINITY;
      tc_before();
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (threadIdx.x == 0) PAIR_TR(5, 2);
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

}  // namespace mtkv_b200

namespace mtkv_b200 {

bool attn_pair_wanted(const PoolGeom& g, const ReqDev* reqs, uint32_t n) {
  static const bool off = [] {  // MTKV_ATTN_PAIR=1 selects the paired kernel (measured variant; default off)
    const char* e = std::getenv("MTKV_ATTN_PAIR");
    return !(e && e[0] == '1');
  }();
  if (off || g.D != 128 || g.S > pair::BN || pair::BN % g.S) return false;
  for (uint32_t r = 0; r < n; ++r)
    if (reqs[r].n_q - reqs[r].q_skip > pair::BM) return true;
  return false;
}

void launch_attention_pair(const CUtensorMap& pool_map, const CUtensorMap& q_map, const AttnArgs& a,
                           cudaStream_t s) {
  if (a.n_items == 0) return;
  static DeviceOnce once;
  if (once.first()) {
    cudaFuncSetAttribute(attn_pair_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pair::SMEM));
    cudaFuncSetAttribute(attn_pair_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pair::SMEM));
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.n_items);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = pair::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (a.trace) cudaLaunchKernelEx(&cfg, attn_pair_kernel<true>, pool_map, q_map, a);
  else cudaLaunchKernelEx(&cfg, attn_pair_kernel<false>, pool_map, q_map, a);
}

}  // namespace mtkv_b200
