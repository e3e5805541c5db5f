// Incremental prefix-reuse attention on the 5th-gen tensor cores (sm_100a).
//
// Persistent kernel: one CTA per SM streams a contiguous, equal-length range
// of 128-key tiles (attn_plan.cpp); the range is a list of pieces, each a key
// range of one (request, head, 128-row query tile) segment. The K/V rings keep
// streaming across piece boundaries, so an SM never idles on a prologue.
// Warp roles (384 threads):
//   warp 0      K producer: page-granular cp.async.bulk.tensor loads of K tiles
//               straight out of the paged pool (no gather pass), NK-stage ring
//   warp 3      V producer: same for V, NV-stage ring (V stays until PV, K is
//               released as soon as S = Q K^T has completed)
//   warp 1      MMA issuer (one elected lane of a uniform warp): tcgen05.cp of
//               the piece's Q into TMEM, S = Q K^T (A = Q in TMEM, B = K in
//               smem) into one of two S buffers, O += P V (A = P in TMEM over
//               its S buffer, B = V in smem) with tcgen05.mma kind::f16
//   warp 2      TMEM allocator, then Q loader (TMA, double-buffered per piece; a
//               buffer is refilled once its Q is in TMEM and the piece's
//               epilogue, which stages O through it, is done)
//   warps 4..11 softmax: thread r of warpgroup w owns query row r (= TMEM lane
//               r) and key columns [64w, 64w + 64) of each tile: tcgen05.ld of
//               its S half, mask, row max exchanged with the other warpgroup
//               through shared memory, online softmax in base 2, P -> TMEM
//               (bf16x2, tcgen05.st over the S buffer), lazy O rescale of its
//               half of O; per piece an epilogue O/l + lse
// While the softmax warps turn S(t) into P(t), the tensor core computes S(t+1)
// into the other buffer; S(t+2) is issued right behind PV(t), which in the
// in-order tensor pipe has read P(t) from the buffer S(t+2) overwrites.
// Logical key space: the user's keys [0, KA) padded to a page boundary, then
// the request's candidate keys (their own scratch pages), so every page-sized
// slice of a tile is one TMA box. Keys past the end load as zeros (TMA OOB).
//
// Shared-memory operand layouts (canonical UMMA, 128-byte swizzle):
//   Q, K : K-major  [rows][64-elem blocks], SBO = 1024 B, +32 B per K=16 step
//   V    : MN-major [keys][64-dim blocks],  SBO = 1024 B, LBO = one block
// TMEM columns: S/P buffers (2 x 128 fp32) | O (D fp32) | Q (D/2).
#include <cuda.h>
#include <cstdio>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>

#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace mtkv_b200 {

namespace tc {

constexpr int BM = 128;   // query rows per tile (TMEM lanes)
constexpr int BN = 128;   // keys per tile (two warpgroups x 64 columns)

#define ATTN_TR(kind, t)                                                                  \
  do {                                                                                    \
    if (TR && blockIdx.x < kTraceCtas && (t) < kTraceTiles)                               \
      a.trace[((size_t)blockIdx.x * kTraceKinds + (kind)) * kTraceTiles + (t)] = gtime(); \
  } while (0)

}  // namespace tc

using namespace tc;


template <int D>
struct TcCfg {
  // 64-element column blocks of Q/K/V. D = 32: one block holding this head and
  // its neighbour (a 128-B swizzled row; the head's operands start SUB bytes
  // into it, which the MMA / tcgen05.cp descriptors address like a K step)
  static constexpr int NB = D >= 64 ? D / 64 : 1;
  static constexpr uint32_t KBLK = BN * 128;             // BN keys x 128 B
  static constexpr uint32_t T_BYTES = NB * KBLK;         // one K (or V, or Q: BM == BN) tile
  static constexpr uint32_t QBLK = KBLK;
  static_assert(BM == BN, "a piece's Q travels through a V ring stage");
#ifndef MTKV_ATTN_NK
#define MTKV_ATTN_NK 4
#endif
  // All shared memory is K/V ring: the more tiles in flight per SM, the more of
  // the loaded DRAM latency (~3 us at full bandwidth, measured) is covered.
  static constexpr int NK = D == 128 ? MTKV_ATTN_NK : 6;      // K ring stages (128-key tiles)
  static constexpr int NV = D == 128 ? 7 - MTKV_ATTN_NK : 6;  // V ring stages (V is held until PV; also carries Q)
  // TMEM: two S buffers (fp32, BN cols; P(t) is written as bf16x2 over the first
  // BN/2 columns of S(t)'s buffer), O (D cols), Q (D/2 cols), L (16 cols: the
  // row sums of P, accumulated by the tensor core as P x ones)
  static constexpr uint32_t S_COL = 0, O_COL = 2 * BN, Q_COL = 2 * BN + D, L_COL = Q_COL + D / 2;
  static constexpr uint32_t TMEM_COLS = L_COL + 16 <= 256 ? 256 : 512;
  static_assert(L_COL + 16 <= 512, "TMEM budget");
  static constexpr size_t SMEM = size_t(NK + NV) * T_BYTES + 2 * 2 * BM * 4 + 128 + 256;
  static_assert(SMEM <= 232448, "shared memory budget");
};

template <int D, bool TR, int POLY>  // TR: per-CTA event trace; POLY: k-th columns use ex2_poly (0: none)
// D in {32, 64, 128}
__global__ void __launch_bounds__(384, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap pool_map, const __grid_constant__ CUtensorMap q_map,
                   AttnArgs a) {
  using C = TcCfg<D>;
  constexpr int NB = C::NB, NK = C::NK, NV = C::NV;
  constexpr uint32_t QBLK = C::QBLK, KBLK = C::KBLK, T_BYTES = C::T_BYTES;
  constexpr int HC = BN / 2;        // key columns per softmax warpgroup
  constexpr float kRescale = 8.f;   // lazy rescale threshold (log2 units): p <= 2^8 between rescales

  extern __shared__ __align__(1024) uint8_t smem_raw[];  // 128-B swizzled tiles need 1024-B alignment
  uint8_t* smem = smem_raw;
  uint8_t* sK = smem;                          // [NK] K tiles
  uint8_t* sV = sK + NK * T_BYTES;             // [NV] V tiles, and each piece's Q ahead of its V tiles
  float* sMax = reinterpret_cast<float*>(sV + NV * T_BYTES);  // [2 tiles][2 warpgroups][BM] row-max exchange
  // 64 bf16 ones: one no-swizzle core matrix (8 rows x 16 B) that the P x ones
  // MMA reads as every core matrix of its [128 keys x 16] B operand (strides 0)
  uint32_t* sOnes = reinterpret_cast<uint32_t*>(sMax + 2 * 2 * BM);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOnes + 32);
  uint64_t* full_k = bars;
  uint64_t* empty_k = full_k + NK;
  uint64_t* full_v = empty_k + NK;
  uint64_t* empty_v = full_v + NV;
  uint64_t* s_full = empty_v + NV;  // [2] S buffer computed
  uint64_t* p_full = s_full + 2;    // P(t) in TMEM + O rescaled (8 softmax warps)
  uint64_t* o_done = p_full + 1;    // PV(t) completed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);

  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const PoolGeom& g = a.g;
  const uint32_t S = g.S;
  if (threadIdx.x == 0) ATTN_TR(5, 0);
  // this CTA's piece range (read ahead of the barrier / TMEM setup)
  const uint32_t pb = a.cta_off[blockIdx.x], pe = a.cta_off[blockIdx.x + 1];

  if (threadIdx.x == 0) {
    // every ring stage is released by the MMA issuer's tcgen05.commit: a K stage
    // once its S = Q K^T completed, a V stage once its PV completed, a Q stage
    // (V ring) once tcgen05.cp moved it into TMEM
    for (int s = 0; s < NK; ++s) { mbar_init(&full_k[s], 1); mbar_init(&empty_k[s], 1); }
    for (int s = 0; s < NV; ++s) { mbar_init(&full_v[s], 1); mbar_init(&empty_v[s], 1); }
    for (int b = 0; b < 2; ++b) mbar_init(&s_full[b], 1);
    mbar_init(p_full, 8);
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) sOnes[threadIdx.x] = 0x3F803F80u;  // bf16x2 (1, 1)
  fence_async_smem();  // visible to the tensor core (async proxy)
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tmem_slot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tmem_slot;
  // Programmatic dependent launch: this grid may start while the projection
  // GEMM that writes Q and appends this layer's fresh K/V is still running.
  // Everything before it in the stream (batch metadata, the cached prefix in the
  // pool, the previous consumer of part_o) is complete, so only reads of Q and
  // of tiles holding fresh keys wait for the GEMM (griddepcontrol.wait below).
  if (threadIdx.x == 0) ATTN_TR(5, 1);
  // the gate/norm kernel (PDL) may be scheduled as CTAs of this grid retire; it
  // waits for the whole grid (griddepcontrol.wait) before reading the partials
  if (a.trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0 || warp == 3) {
    // ---------------- K / V producers (whole warp: lane i resolves page i) ----------------
    // The V ring also carries each piece's Q tile, loaded right ahead of the
    // piece's first V tile (Q is written by the projection GEMM: the V producer
    // waits for it up front; V is consumed a softmax pass after K anyway, so
    // only the K producer streams cached-prefix tiles before the GEMM retires).
    const bool isv = warp == 3;
    uint64_t* full = isv ? full_v : full_k;
    uint64_t* empty = isv ? empty_v : empty_k;
    uint8_t* ring = isv ? sV : sK;
    const uint32_t NS = isv ? NV : NK;
    const uint32_t ppt = BN / S;  // pages per tile
    uint32_t gt = 0, st = 0, ph = 0;
    bool dep_done = false;        // griddepcontrol.wait executed
    if (isv) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      dep_done = true;
    }
    auto acquire = [&]() -> uint8_t* {  // lane 0: wait for the next stage and arm it for one tile
      if (lane == 0) {
        if (gt >= NS) mbar_wait(&empty[st], ph ^ 1);
        mbar_expect_tx(&full[st], T_BYTES);
      }
      __syncwarp();
      return ring + st * T_BYTES;
    };
    auto advance = [&]() {
      ++gt;
      if (++st == NS) { st = 0; ph ^= 1; }
    };
    for (uint32_t pc = pb; pc < pe; ++pc) {
      const AttnPiece P = a.pieces[pc];
      const uint64_t KA = P.start + P.n_hist;
      const uint32_t user_pages = uint32_t((KA + S - 1) / S);
      const uint32_t col = (P.head * D) & ~63u;  // first 64-column block of this head
      auto row_of = [&](uint64_t lp) -> int {  // pool row of a logical page's K slice
        uint32_t page;
        if (lp < user_pages) page = a.pages[P.pages_off + uint32_t(lp)];
        else if (lp - user_pages < P.n_scratch && (lp - user_pages) * S < P.n_cand)
          page = a.pages[P.scratch_off + uint32_t(lp - user_pages)];
        else return -int(S) * 4;  // out of bounds -> TMA zero fill
        return int(((uint64_t(a.layer) * g.num_pages + page) * 2) * S);
      };
      if (isv) {  // the piece's Q (one TMA box per 64-column block)
        uint8_t* dst = acquire();
        if (lane == 0) {
#pragma unroll
          for (int b = 0; b < NB; ++b)
            tma_load_2d(dst + b * QBLK, &q_map, int(col + 64 * b), int(P.q_row0 + P.q_skip + P.qtile * BM), &full[st]);
        }
        advance();
      }
      uint32_t cache_t0 = P.lo;
      int rows_cache = row_of(uint64_t(P.lo) * ppt + lane);  // 32 consecutive pages per refresh
      for (uint32_t t = P.lo; t < P.hi; ++t) {
        if ((t - cache_t0) * ppt >= 32) {
          cache_t0 = t;
          rows_cache = row_of(uint64_t(t) * ppt + lane);
        }
        if (!dep_done && uint64_t(t + 1) * BN > P.dep_start) {  // tile holds keys this layer's GEMM appends
          asm volatile("griddepcontrol.wait;" ::: "memory");
          dep_done = true;
        }
        if (!isv && lane == 0) ATTN_TR(0, gt);
        uint8_t* dst = acquire();
        for (uint32_t i = 0; i < ppt; ++i) {
          int row = __shfl_sync(0xffffffffu, rows_cache, (t - cache_t0) * ppt + i);
          if (isv && row >= 0) row += int(S);
          if (lane == 0) {
#pragma unroll
            for (int b = 0; b < NB; ++b)
              tma_load_2d(dst + b * KBLK + i * S * 128, &pool_map, int(col + 64 * b), row, &full[st]);
          }
        }
        advance();
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // Order: S(0), S(1), then per tile t: PV(t) (waits for P(t)), S(t+2) into
    // S(t)'s buffer — in order behind PV(t), which has read P(t) from it. S(t+1)
    // runs on the tensor core while the softmax warps turn S(t) into P(t).
    // The whole warp runs branch-free uniform code; one elected lane issues.
    if (pe > pb) {
      constexpr uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
      constexpr uint32_t idesc_o =
          (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(D >> 3) << 17) | (uint32_t(BM >> 4) << 24);
      // row sums: L[128 x 16] += P[128 x 128 keys] x ones[128 x 16] (B K-major, no swizzle, all strides 0)
      constexpr uint32_t idesc_l = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(16 >> 3) << 17) | (uint32_t(BM >> 4) << 24);
      const uint64_t d_ones = uint64_t((s32(sOnes) >> 4) & 0x3FFF) | (uint64_t(1) << 46);
      const uint64_t dk0 = sdesc(s32(sK), 16, 1024), dq0 = sdesc(s32(sV), 16, 1024), dv0 = sdesc(s32(sV), KBLK, 1024);
      const bool leader = elect_one();
      uint32_t total = 0;
      for (uint32_t pc = pb; pc < pe; ++pc) total += a.pieces[pc].hi - a.pieces[pc].lo;
      // S cursor
      uint32_t s_pc = pb, s_left = a.pieces[pb].hi - a.pieces[pb].lo, s_j = 0, stk = 0, phk = 0, s_g = 0;
      uint32_t s_sub = 0;  // D = 32: byte offset of the piece's head inside its 64-column block
      // V-ring positions: the producer fills the ring as Q(p), V tiles of p,
      // Q(p+1), ... S runs two tiles ahead of PV, so Q(p+1) is taken (by the
      // piece's first S) before the last V tiles of p: each side keeps its own
      // position (stage = pos % NV, phase = pos / NV), stages are released out
      // of order by their own commits
      uint32_t pv_pc = pb, pv_left = a.pieces[pb].hi - a.pieces[pb].lo;  // PV-side piece cursor
      uint32_t pv_next = 1;  // V-ring position of the next V tile (Q(pb) sits at 0)
      uint32_t q_next = 0;   // V-ring position of the next piece's Q
      auto issue_s = [&]() {
        const uint32_t b = s_g & 1;
        ATTN_TR(9, s_g);
        if (s_j == 0) {
          // new piece: copy its Q (V ring) into TMEM, in order behind the
          // previous piece's S MMAs that still read the old Q
          const uint32_t qs = q_next % NV, qph = (q_next / NV) & 1;
          s_sub = D < 64 ? ((a.pieces[s_pc].head * D) & 63u) * 2 : 0;
          mbar_wait(&full_v[qs], qph);
          tc_after();
          const uint64_t aq = dq0 + ((qs * T_BYTES + s_sub) >> 4);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            tmem_cp_if(leader, tmem + C::Q_COL + kk * 8, aq + ((((kk / 4) * QBLK + (kk % 4) * 32)) >> 4));
          mma_commit_if(leader, &empty_v[qs]);  // stage reusable once copied
          // the following piece's Q sits after this piece's Q and V tiles
          q_next += 1 + (a.pieces[s_pc].hi - a.pieces[s_pc].lo);
        }
        mbar_wait(&full_k[stk], phk);
        tc_after();
        const uint64_t bk = dk0 + ((stk * T_BYTES + s_sub) >> 4);
        const uint32_t d_tmem = tmem + C::S_COL + b * BN;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ts_if(leader, d_tmem, tmem + C::Q_COL + kk * 8, bk + (((kk / 4) * KBLK + (kk % 4) * 32) >> 4), idesc_s,
                    kk > 0);
        mma_commit_if(leader, &s_full[b]);
        mma_commit_if(leader, &empty_k[stk]);  // K stage read once S completed
        if (leader) ATTN_TR(1, s_g);
        if (++stk == NK) { stk = 0; phk ^= 1; }
        ++s_g;
        ++s_j;
        if (--s_left == 0) {
          ++s_pc;
          s_j = 0;
          if (s_pc < pe) { const AttnPiece Pn = a.pieces[s_pc]; s_left = Pn.hi - Pn.lo; }
        }
      };
      issue_s();
      if (s_g < total) issue_s();
      uint32_t v_j = 0;
      for (uint32_t gg = 0; gg < total; ++gg) {
        ATTN_TR(10, gg);
        const uint32_t stv = pv_next % NV, phv = (pv_next / NV) & 1;
        mbar_wait(p_full, gg & 1);
        mbar_wait(&full_v[stv], phv);
        tc_after();
        const uint32_t v_sub = D < 64 ? ((a.pieces[pv_pc].head * D) & 63u) * 2 : 0;
        const uint64_t bv = dv0 + ((stv * T_BYTES + v_sub) >> 4);
        const uint32_t a_tmem = tmem + C::S_COL + (gg & 1) * BN;  // P(gg) over S(gg)'s buffer
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          mma_ts_if(leader, tmem + C::O_COL, a_tmem + kk * 8, bv + ((kk * 2048) >> 4), idesc_o,
                    (v_j > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          mma_ts_if(leader, tmem + C::L_COL, a_tmem + kk * 8, d_ones, idesc_l, (v_j > 0 || kk > 0) ? 1u : 0u);
        mma_commit_if(leader, o_done);
        mma_commit_if(leader, &empty_v[stv]);  // V stage read once PV completed
        if (leader) ATTN_TR(2, gg);
        ++pv_next;
        ++v_j;
        if (--pv_left == 0) {
          ++pv_pc;
          v_j = 0;
          ++pv_next;  // skip the next piece's Q
          if (pv_pc < pe) { const AttnPiece Pn = a.pieces[pv_pc]; pv_left = Pn.hi - Pn.lo; }
        }
        if (s_g < total) issue_s();
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax: 8 warps, warpgroup w takes key columns [w*BN/2, (w+1)*BN/2) ----------------
    const uint32_t wg = (warp - 4) / 4;            // column half
    const uint32_t r = (threadIdx.x - 128) % 128;  // query row == TMEM lane
    const uint32_t lane_base = (32u * (warp % 4)) << 16;
    const uint32_t o_col = tmem + lane_base + C::O_COL + wg * (D / 2);
    uint32_t t_all = 0;      // tiles processed (barrier phases)
    auto named_sync = [&]() { asm volatile("bar.sync 1, 256;" ::: "memory"); };
    // A piece's epilogue (O / l and lse into its slot) is deferred into the next
    // piece's first tile, after that tile's exponentials and before its P is
    // released: the wait for the piece's last PV then overlaps softmax work, and
    // O / L are still read before the next piece's first PV (issued after that
    // p_full) overwrites them. The CTA's last piece is written after the loop.
    bool ep_pend = false, ep_valid = false;
    uint32_t ep_part = 0, ep_pc = 0;
    float ep_mref = 0.f;
    auto epilogue = [&]() {  // the pending piece's last PV has completed
      if (threadIdx.x == 128) ATTN_TR(11, 4 * (ep_pc - pb));
      // O/l straight from TMEM to the slot: thread r owns row r's D/2 columns of
      // this half; in the chunked slot layout (part_index) a warp's store of
      // one 4-column chunk covers 32 consecutive rows = 512 contiguous bytes.
      // Rows past the tile's valid rows are not written (the combine never
      // reads them). L and this half of O are loaded with one wait.
      constexpr int OC = D / 2;  // O columns of this half
      float o[OC];
      const float l_run = tmem_ld1(tmem + lane_base + C::L_COL);  // row sum of P (all 16 columns equal)
      if constexpr (OC >= 32) {
#pragma unroll
        for (int c = 0; c < OC / 32; ++c) tmem_ld32(o_col + c * 32, o + c * 32);
      } else {
        tmem_ld16(o_col, o);
      }
      tmem_wait_ld();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      if (threadIdx.x == 128) ATTN_TR(11, 4 * (ep_pc - pb) + 1);
      float* dst = a.part_o + part_index(ep_part, BM, r, wg * (D / 2), D);
      constexpr size_t chunk_stride = size_t(BM) * 4;  // floats between consecutive 4-column chunks
      if (ep_valid) {
#pragma unroll
        for (int k = 0; k < OC / 4; ++k)
          *reinterpret_cast<float4*>(dst + k * chunk_stride) =
              make_float4(o[4 * k] * inv, o[4 * k + 1] * inv, o[4 * k + 2] * inv, o[4 * k + 3] * inv);
      }
      if (wg == 0 && ep_valid) a.part_lse[size_t(ep_part) * BM + r] = l_run > 0.f ? ep_mref + log2f(l_run) : -INFINITY;
      if (threadIdx.x == 128) ATTN_TR(5, 4 + 2 * (ep_pc - pb));
      ep_pend = false;
    };
    for (uint32_t pc = pb; pc < pe; ++pc) {
      const AttnPiece P = a.pieces[pc];
      const uint64_t KA = P.start + P.n_hist;
      const uint64_t KAp = (KA + S - 1) / S * S;
      const uint32_t q0 = P.q_skip + P.qtile * BM;
      const uint32_t q_end = min(P.n_q, q0 + BM);
      const uint64_t pos_last = P.start + q_end - 1;
      const uint64_t k_vis = pos_last >= KA ? KAp + (pos_last - KA + 1) : pos_last + 1;
      const uint64_t k_hi = min(k_vis, uint64_t(P.hi) * BN);
      const uint64_t pos_r = P.start + q0 + r;
      // valid keys of this row: user keys [0, u_end), candidate keys [KAp, c_end)
      const uint64_t u_end = min(min(KA, k_hi), pos_r + 1);
      const uint64_t c_end = pos_r >= KA ? min(min(KAp + P.n_cand, KAp + (pos_r - KA + 1)), k_hi) : KAp;
      // the same bounds relative to this warpgroup's first key of the piece, clamped (32-bit per tile)
      const uint64_t kb0 = uint64_t(P.lo) * BN + wg * HC;
      const int64_t span = int64_t(P.hi - P.lo) * BN;
      auto rel = [&](uint64_t x) { return int(min(max(int64_t(x) - int64_t(kb0), int64_t(-1)), span)); };
      const int ue = rel(u_end), cl = rel(KAp), ce = rel(c_end);
      float m_ref = -INFINITY;
      for (uint32_t t = P.lo; t < P.hi; ++t, ++t_all) {
        const uint32_t b = t_all & 1;
        mbar_wait(&s_full[b], (t_all >> 1) & 1);
        tc_after();
        if (threadIdx.x % 128 == 0) ATTN_TR(3, t_all);
        float s[HC];
#pragma unroll
        for (int c = 0; c < HC / 32; ++c) tmem_ld32(tmem + lane_base + C::S_COL + b * BN + wg * HC + c * 32, s + c * 32);
        tmem_wait_ld();
        const int kb = int(t - P.lo) * BN;
        const int cu = min(max(ue - kb, 0), HC), c_lo = min(max(cl - kb, 0), HC), c_hi = min(max(ce - kb, 0), HC);
        if (cu != HC) {
          // valid columns as a bit mask per 32-column chunk: one shift + select per
          // element (a per-element || compiled to a divergent branch each)
#pragma unroll
          for (int q = 0; q < (HC + 31) / 32; ++q) {
            const int c0 = q * 32;
            const uint32_t bits = range_bits(-c0, cu - c0) | range_bits(c_lo - c0, c_hi - c0);
#pragma unroll
            for (int c = 0; c < 32 && c0 + c < HC; ++c) s[c0 + c] = (bits >> c) & 1u ? s[c0 + c] : -INFINITY;
          }
        }
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < HC; ++c) m4[c & 3] = fmaxf(m4[c & 3], s[c]);
        // row max over both halves: exchange through shared memory (double-buffered by tile)
        float* mx_buf = sMax + b * 2 * BM;
        mx_buf[wg * BM + r] = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        named_sync();  // also orders both halves' S loads before either writes P over them
        const float mx = fmaxf(mx_buf[r], mx_buf[BM + r]) * a.scale_log2;
        if (threadIdx.x % 128 == 0) ATTN_TR(6, t_all);
        float alpha = 1.f;
        if (mx > m_ref + kRescale) {
          alpha = m_ref == -INFINITY ? 0.f : ex2(m_ref - mx);
          m_ref = mx;
        }
        const float nmref = m_ref == -INFINITY ? 0.f : -m_ref;
        // (the row sum of P is accumulated by the tensor core: L += P x ones)
#pragma unroll
        for (int c = 0; c < HC; ++c) {
          const float x = fmaf(s[c], a.scale_log2, nmref);
          s[c] = (POLY && c % POLY == POLY - 1) ? ex2_poly(x) : ex2(x);
        }
        if (threadIdx.x % 128 == 0) ATTN_TR(7, t_all);
        // P over the first BN/2 columns of this S buffer (this half's HC/2 columns)
#pragma unroll
        for (int hlf = 0; hlf < HC / 32; ++hlf) {
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) pk[c] = pack2(s[hlf * 32 + 2 * c], s[hlf * 32 + 2 * c + 1]);
          tmem_st16(tmem + lane_base + C::S_COL + b * BN + wg * (HC / 2) + hlf * 16, pk);
        }
        if (t != P.lo) {  // the previous PV must finish before O is rescaled
          mbar_wait(o_done, (t_all - 1) & 1);
          tc_after();
          if (__any_sync(0xffffffffu, alpha != 1.f)) {
            if (wg == 0) tmem_st1(tmem + lane_base + C::L_COL, tmem_ld1(tmem + lane_base + C::L_COL) * alpha);
            if constexpr (D >= 64) {
#pragma unroll 1
              for (int c = 0; c < D / 64; ++c) {
                float o[32];
                tmem_ld32(o_col + c * 32, o);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) o[i] *= alpha;
                tmem_st32(o_col + c * 32, o);
              }
            } else {  // D = 32: 16 O columns per warpgroup
              float o[16];
              tmem_ld16(o_col, o);
              tmem_wait_ld();
              uint32_t w[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) w[i] = __float_as_uint(o[i] * alpha);
              tmem_st16(o_col, w);
            }
          }
        } else if (ep_pend) {  // the previous piece's epilogue (its last PV is tile t_all - 1)
          if (threadIdx.x == 128) ATTN_TR(5, 3 + 2 * (ep_pc - pb));
          mbar_wait(o_done, (t_all - 1) & 1);
          tc_after();
          epilogue();
        }
        if (threadIdx.x % 128 == 0) ATTN_TR(8, t_all);
        tmem_wait_st();
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        if (threadIdx.x % 128 == 0) ATTN_TR(4, t_all);
      }
      // ---- epilogue (O / l and lse into slot P.part): deferred, see above ----
      ep_pend = true;
      ep_part = P.part;
      ep_valid = q0 + r < q_end;
      ep_mref = m_ref;
      ep_pc = pc;
    }
    if (ep_pend) {  // the CTA's last piece
      if (threadIdx.x == 128) ATTN_TR(5, 3 + 2 * (ep_pc - pb));
      mbar_wait(o_done, (t_all - 1) & 1);
      tc_after();
      epilogue();
      tc_before();
    }
    if (threadIdx.x == 128) ATTN_TR(5, 2);
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
}

// ------------------------------------------------------------------ host ---
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn), cudaEnableDefault, &q);
  }
  return fn;
}

// D = 32 reads 64-column blocks (two heads): the hidden width must be a whole
// number of blocks so the TMA boxes stay inside a row
bool attn_tc_supported(const PoolGeom& g) {
  return (g.D == 64 || g.D == 128 || (g.D == 32 && g.d % 64 == 0)) && g.S >= 8 && g.S <= BN && (BN % g.S) == 0;
}

int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 1;
}

static int encode_2d(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  auto fn = encode_fn();
  if (!fn) return -1;
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

// pool viewed as rows of d elements: [L * num_pages * 2 * S][d], box = 64 cols x one page
int make_pool_map(CUtensorMap* map, const void* pool, const PoolGeom& g) {
  return encode_2d(map, pool, g.d, uint64_t(g.L) * g.num_pages * 2 * g.S, g.S);
}

// fresh-row queries [rows][d], box = 64 cols x 128 rows (rows past the buffer load as zeros)
int make_q_map(CUtensorMap* map, const void* q, uint64_t rows, const PoolGeom& g) {
  return encode_2d(map, q, g.d, rows, BM);
}

template <int D, bool TR, int POLY>
static void launch_cfg(const CUtensorMap& pool_map, const CUtensorMap& q_map,
                       const AttnArgs& a, cudaStream_t s) {
  static DeviceOnce once;
  if (once.first())
    cudaFuncSetAttribute(attn_tc_kernel<D, TR, POLY>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(TcCfg<D>::SMEM));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.n_items);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = TcCfg<D>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL: prologue overlaps the GEMM's tail
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, attn_tc_kernel<D, TR, POLY>, pool_map, q_map, a);
}

template <int D>
static void launch_tc_d(const CUtensorMap& pool_map, const CUtensorMap& q_map,
                        const AttnArgs& a, cudaStream_t s) {
  static const int poly = [] {
    const char* e = std::getenv("MTKV_ATTN_POLY");
    return e ? std::atoi(e) : kPolyDefault;
  }();
  if (a.trace) launch_cfg<D, true, kPolyDefault>(pool_map, q_map, a, s);
  else if (poly == 2) launch_cfg<D, false, 2>(pool_map, q_map, a, s);
  else if (poly == 3) launch_cfg<D, false, 3>(pool_map, q_map, a, s);
  else if (poly == 4) launch_cfg<D, false, 4>(pool_map, q_map, a, s);
  else if (poly == 8) launch_cfg<D, false, 8>(pool_map, q_map, a, s);
  else launch_cfg<D, false, 0>(pool_map, q_map, a, s);
}

void launch_attention_tc(const CUtensorMap& pool_map, const CUtensorMap& q_map,
                         const AttnArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return;
  static const bool no_trigger = [] {  // MTKV_ATTN_TRIGGER=0: A/B switch for the early PDL release
    const char* e = std::getenv("MTKV_ATTN_TRIGGER");
    return e && e[0] == '0';
  }();
  AttnArgs b = a;
  if (no_trigger) b.trigger = 0;
  if (a.g.D == 32) launch_tc_d<32>(pool_map, q_map, b, s);
  else if (a.g.D == 64) launch_tc_d<64>(pool_map, q_map, b, s);
  else launch_tc_d<128>(pool_map, q_map, b, s);
}

}  // namespace mtkv_b200
