// Incremental prefix-reuse attention, two-lane form (sm_100a).
//
// Same work decomposition as attn_tc.cu (pieces = ranges of 128-key plan tiles
// of (request, head, 128-row query tile) segments), planned over 2 x SMs
// virtual CTAs: each persistent CTA runs TWO independent pipelines ("lanes"),
// lane X = virtual CTA 2b + X (with the head-sibling plan: the two heads of the
// same rows, i.e. the two column halves of the same pool rows). A lane has its
// own producer warp, MMA warp, K/V rings, Q tile (shared memory), double-
// buffered S and an O accumulator (TMEM), and a softmax warpgroup in which
// thread r owns query row r and every key column of a 64-key sub-tile (no
// cross-warpgroup max exchange). The lanes share only the SM: while one lane's
// warpgroup turns S into P on the MUFU/FMA pipes, the other's MMAs run on the
// tensor core, and each lane's stalls (piece boundaries, epilogues, rescales)
// are covered by the other lane's work. (The column-split form, attn_tc.cu,
// runs one 128-key tile at a time with both warpgroups in lockstep, so the
// MUFU idles during every max exchange, P store and epilogue.)
// Per lane, S(u+1) is computed while the softmax works on S(u); S(u+2) is
// issued right behind PV(u) into S(u)'s buffer.
// 64-key sub-tiles keep TMEM at 2 x (2 S x 64 + O D) <= 512 columns.
// Warps (384 threads):
//   0 / 3   producer of lane A / B: Q at each piece start (once the piece
//           before has no S left to issue), K and V sub-tiles
//   1 / 2   MMA issuer of lane A / B (warp 2 also allocates TMEM)
//   4..7    softmax + epilogue of lane A
//   8..11   softmax + epilogue of lane B
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <string>

#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace mtkv_b200 {

using namespace tc;

namespace pp {
constexpr int BM = 128;   // query rows per tile (TMEM lanes)
constexpr int PT = 128;   // keys per plan tile (attn_plan.cpp kTcBN)
constexpr int BN = 64;    // keys per sub-tile

template <int D>
struct Cfg {
  static constexpr int NB = D / 64;                     // 64-column blocks of Q / K / V
  static constexpr uint32_t KBLK = BN * 128;            // BN keys x 128 B
  static constexpr uint32_t T_BYTES = NB * KBLK;        // one K or V sub-tile
  static constexpr uint32_t QBLK = BM * 128;            // 128 rows x 128 B
  static constexpr uint32_t Q_BYTES = NB * QBLK;        // one lane's Q
  static constexpr int NK = D == 128 ? 3 : 6;           // K ring stages per lane
  static constexpr int NV = D == 128 ? 2 : 5;           // V ring stages per lane
  // TMEM per lane x: S buffers [x*2BN, x*2BN + 2BN) (P as bf16x2 over a buffer's
  // first BN/2 columns), O at 4BN + x*D
  static constexpr uint32_t O_COL = 4 * BN;
  static constexpr uint32_t TMEM_COLS = 512;
  static_assert(O_COL + 2 * D <= TMEM_COLS, "TMEM budget");
  static constexpr uint32_t LANE_SMEM = Q_BYTES + (NK + NV) * T_BYTES;
  static constexpr uint32_t NBAR = 2 * NK + 2 * NV + 6;  // per lane
  static constexpr size_t SMEM = 2 * size_t(LANE_SMEM) + 2 * NBAR * 8 + 16;
  static_assert(SMEM <= 232448, "shared memory budget");
};
}  // namespace pp

// MTKV_ATTN_TRACE: lane A's event times (kinds as in tools/attn_trace_stats.py:
// 0 K issued, 9 V issued, 1 S issued, 10 PV: P ready, 11 PV: V ready, 2 PV
// issued, 3 S ready (softmax), 6 S loaded + max, 7 exps done, 4 P arrived,
// 5 [0] start [1] setup [2] end [3+2k, 4+2k] epilogue k)
#define PP_TR(kind, t)                                                                    \
  do {                                                                                    \
    if (TR && x == 0 && blockIdx.x < kTraceCtas && (t) < kTraceTiles)                     \
      a.trace[((size_t)blockIdx.x * kTraceKinds + (kind)) * kTraceTiles + (t)] = gtime(); \
  } while (0)

template <int D, bool TR>
__global__ void __launch_bounds__(384, 1)
    attn_pp_kernel(const __grid_constant__ CUtensorMap pool_map, const __grid_constant__ CUtensorMap q_map,
                   AttnArgs a) {
  using namespace pp;
  using C = Cfg<D>;
  constexpr int NB = C::NB, NK = C::NK, NV = C::NV;
  constexpr uint32_t KBLK = C::KBLK, T_BYTES = C::T_BYTES, QBLK = C::QBLK, Q_BYTES = C::Q_BYTES;
  constexpr float kRescale = 8.f;  // lazy rescale threshold (log2 units)

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // lane of this warp: producers 0 / 3, MMA 1 / 2, softmax 4-7 / 8-11
  const uint32_t x = warp >= 4 ? (warp - 4) / 4 : (warp == 0 || warp == 1) ? 0u : 1u;
  uint8_t* sQ = smem_raw + x * C::LANE_SMEM;   // this lane's Q
  uint8_t* sK = sQ + Q_BYTES;                  // [NK]
  uint8_t* sV = sK + NK * T_BYTES;             // [NV]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + 2 * C::LANE_SMEM) + x * C::NBAR;
  uint64_t* full_k = bars;
  uint64_t* empty_k = full_k + NK;
  uint64_t* full_v = empty_k + NK;
  uint64_t* empty_v = full_v + NV;
  uint64_t* q_full = empty_v + NV;   // Q landed
  uint64_t* q_free = q_full + 1;     // the piece's last S completed (Q no longer read)
  uint64_t* s_full = q_free + 1;     // [2] S buffer computed
  uint64_t* p_full = s_full + 2;     // P in TMEM (+ O rescaled): 4 softmax warps
  uint64_t* o_done = p_full + 1;     // PV completed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(reinterpret_cast<uint64_t*>(smem_raw + 2 * C::LANE_SMEM) + 2 * C::NBAR);

  const PoolGeom& g = a.g;
  const uint32_t S = g.S;
  const uint32_t pb = a.cta_off[2 * blockIdx.x + x], pe = a.cta_off[2 * blockIdx.x + x + 1];
  if (threadIdx.x == 0) PP_TR(5, 0);

  if (threadIdx.x == 0) {
    for (int xx = 0; xx < 2; ++xx) {
      uint64_t* b = reinterpret_cast<uint64_t*>(smem_raw + 2 * C::LANE_SMEM) + xx * C::NBAR;
      for (int s = 0; s < NK; ++s) { mbar_init(&b[s], 1); mbar_init(&b[NK + s], 1); }
      for (int s = 0; s < NV; ++s) { mbar_init(&b[2 * NK + s], 1); mbar_init(&b[2 * NK + NV + s], 1); }
      uint64_t* q = b + 2 * NK + 2 * NV;
      mbar_init(&q[0], 1);  // q_full
      mbar_init(&q[1], 1);  // q_free
      mbar_init(&q[2], 1);  // s_full[0]
      mbar_init(&q[3], 1);  // s_full[1]
      mbar_init(&q[4], 4);  // p_full
      mbar_init(&q[5], 1);  // o_done
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tmem_slot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) PP_TR(5, 1);
  if (a.trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t s_base = x * 2 * BN, o_base = C::O_COL + x * D;

  if (warp == 0 || warp == 3) {
    // ---------------- producer of lane x ----------------
    // thread 0: the piece's Q (once the piece before has no S left) and the K
    // sub-tiles; thread 1: the V sub-tiles. Independent loops (each blocks only
    // on its own ring), so K streams ahead of V by the K ring's depth.
    if (lane < 2) {
      const bool isv = lane == 1;
      const uint32_t NS = isv ? NV : NK;
      uint64_t* full = isv ? full_v : full_k;
      uint64_t* empty = isv ? empty_v : empty_k;
      uint8_t* ring = isv ? sV : sK;
      const uint32_t pps = BN / S;  // pages per sub-tile (<= 8)
      uint32_t gt = 0;
      bool dep_done = false;
      for (uint32_t pc = pb; pc < pe; ++pc) {
        const AttnPiece P = a.pieces[pc];
        const uint64_t KA = P.start + P.n_hist;
        const uint32_t user_pages = uint32_t((KA + S - 1) / S);
        const uint32_t col = P.head * D;
        auto row_of = [&](uint32_t lp) -> int {  // pool row of a logical page's K (or V) slice
          uint32_t page;
          if (lp < user_pages) page = a.pages[P.pages_off + lp];
          else if (lp - user_pages < P.n_scratch && (lp - user_pages) * S < P.n_cand)
            page = a.pages[P.scratch_off + lp - user_pages];
          else return -int(S) * 4;  // out of bounds -> TMA zero fill
          return int(((uint64_t(a.layer) * g.num_pages + page) * 2 + (isv ? 1 : 0)) * S);
        };
        if (!isv) {  // Q (written by the projection GEMM)
          if (!dep_done) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            dep_done = true;
          }
          if (pc > pb) mbar_wait(q_free, (pc - pb - 1) & 1);
          mbar_expect_tx(q_full, Q_BYTES);
#pragma unroll
          for (int b = 0; b < NB; ++b)
            tma_load_2d(sQ + b * QBLK, &q_map, int(col + 64 * b), int(P.q_row0 + P.qtile * BM), q_full);
        }
        int rows[8], nxt[8];
        for (uint32_t i = 0; i < pps; ++i) nxt[i] = row_of(2 * P.lo * pps + i);
        for (uint32_t u = 2 * P.lo; u < 2 * P.hi; ++u) {
          for (uint32_t i = 0; i < pps; ++i) rows[i] = nxt[i];
          if (!dep_done && uint64_t(u + 1) * BN > P.dep_start) {  // holds keys this layer's GEMM appends
            asm volatile("griddepcontrol.wait;" ::: "memory");
            dep_done = true;
          }
          if (u + 1 < 2 * P.hi)  // the next sub-tile's page rows load while this one waits for a stage
            for (uint32_t i = 0; i < pps; ++i) nxt[i] = row_of((u + 1) * pps + i);
          const uint32_t st = gt % NS;
          if (gt >= NS) mbar_wait(&empty[st], ((gt / NS) & 1) ^ 1);
          PP_TR(isv ? 9 : 0, gt);
          mbar_expect_tx(&full[st], T_BYTES);
          uint8_t* dst = ring + st * T_BYTES;
          for (uint32_t i = 0; i < pps; ++i)
#pragma unroll
            for (int b = 0; b < NB; ++b) tma_load_2d(dst + b * KBLK + i * S * 128, &pool_map, int(col + 64 * b), rows[i], &full[st]);
          ++gt;
        }
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ---------------- MMA issuer of lane x ----------------
    // per piece: S(0), S(1), then per sub-tile u: PV(u) (waits P(u)), S(u+2) into
    // S(u)'s buffer — in order behind PV(u), which has read P(u) from it
    constexpr uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
    constexpr uint32_t idesc_o =
        (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(D >> 3) << 17) | (uint32_t(BM >> 4) << 24);
    const uint64_t dq0 = sdesc(s32(sQ), 16, 1024), dk0 = sdesc(s32(sK), 16, 1024), dv0 = sdesc(s32(sV), KBLK, 1024);
    const bool leader = elect_one();
    uint32_t ns = 0, npv = 0;  // S / PV issued (lane-wide counts: ring positions, barrier phases)
    for (uint32_t pc = pb; pc < pe; ++pc) {
      const AttnPiece P = a.pieces[pc];
      const uint32_t n = 2 * (P.hi - P.lo);  // sub-tiles of the piece
      mbar_wait(q_full, (pc - pb) & 1);
      tc_after();
      auto issue_s = [&](uint32_t j) {  // S of the piece's sub-tile j
        const uint32_t st = ns % NK, b = ns & 1;
        mbar_wait(&full_k[st], (ns / NK) & 1);
        tc_after();
        const uint64_t bk = dk0 + ((st * T_BYTES) >> 4);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = ((kk / 4) * KBLK + (kk % 4) * 32) >> 4;
          const uint32_t qoff = ((kk / 4) * QBLK + (kk % 4) * 32) >> 4;
          asm volatile(
              "{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nsetp.ne.b32 q, %5, 0;\n"
              "@q tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + s_base + b * BN),
              "l"(dq0 + qoff), "l"(bk + off), "r"(idesc_s), "r"(uint32_t(kk > 0)), "r"(uint32_t(leader))
              : "memory");
        }
        mma_commit_if(leader, &s_full[b]);
        mma_commit_if(leader, &empty_k[st]);
        if (leader) PP_TR(1, ns);
        if (j + 1 == n) mma_commit_if(leader, q_free);  // the piece's Q is no longer read
        ++ns;
      };
      issue_s(0);
      if (n > 1) issue_s(1);
      for (uint32_t j = 0; j < n; ++j) {
        const uint32_t st = npv % NV;
        mbar_wait(p_full, npv & 1);
        if (leader) PP_TR(10, npv);
        mbar_wait(&full_v[st], (npv / NV) & 1);
        if (leader) PP_TR(11, npv);
        tc_after();
        const uint64_t bv = dv0 + ((st * T_BYTES) >> 4);
        const uint32_t a_tmem = tmem + s_base + (npv & 1) * BN;  // P(u) over S(u)'s buffer
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          mma_ts_if(leader, tmem + o_base, a_tmem + kk * 8, bv + ((kk * 2048) >> 4), idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit_if(leader, o_done);
        mma_commit_if(leader, &empty_v[st]);
        if (leader) PP_TR(2, npv);
        ++npv;
        if (j + 2 < n) issue_s(j + 2);
      }
    }
  } else {
    // ---------------- softmax + epilogue of lane x ----------------
    const uint32_t r = threadIdx.x % 128;             // query row == TMEM lane
    const uint32_t lane_base = (32u * (warp % 4)) << 16;
    const uint32_t o_col = tmem + lane_base + o_base;
    uint32_t n_all = 0;  // sub-tiles processed (barrier phases)
    for (uint32_t pc = pb; pc < pe; ++pc) {
      const AttnPiece P = a.pieces[pc];
      const uint64_t KA = P.start + P.n_hist;
      const uint64_t KAp = (KA + S - 1) / S * S;
      const uint32_t q0 = P.qtile * BM;
      const uint32_t q_end = min(P.n_q, q0 + BM);
      const uint64_t pos_last = P.start + q_end - 1;
      const uint64_t k_vis = pos_last >= KA ? KAp + (pos_last - KA + 1) : pos_last + 1;
      const uint64_t k_hi = min(k_vis, uint64_t(P.hi) * PT);
      const uint64_t pos_r = P.start + q0 + r;
      // valid keys of this row: user keys [0, u_end), candidate keys [KAp, c_end)
      const uint64_t u_end = min(min(KA, k_hi), pos_r + 1);
      const uint64_t c_end = pos_r >= KA ? min(min(KAp + P.n_cand, KAp + (pos_r - KA + 1)), k_hi) : KAp;
      const uint64_t kb0 = uint64_t(P.lo) * PT;
      const int64_t span = int64_t(P.hi - P.lo) * PT;
      auto rel = [&](uint64_t v) { return int(min(max(int64_t(v) - int64_t(kb0), int64_t(-1)), span)); };
      const int ue = rel(u_end), cl = rel(KAp), ce = rel(c_end);
      float m_ref = -INFINITY, l_run = 0.f;
      for (uint32_t u = 2 * P.lo; u < 2 * P.hi; ++u, ++n_all) {
        const uint32_t b = n_all & 1;
        const uint32_t s_col = tmem + lane_base + s_base + b * BN;
        mbar_wait(&s_full[b], (n_all >> 1) & 1);
        tc_after();
        if (threadIdx.x % 128 == 0) PP_TR(3, n_all);
        float v[BN];
        tmem_ld32(s_col, v);
        tmem_ld32(s_col + 32, v + 32);
        tmem_wait_ld();
        const int kb = int(u - 2 * P.lo) * BN;
        const int cu = min(max(ue - kb, 0), BN), c_lo = min(max(cl - kb, 0), BN), c_hi = min(max(ce - kb, 0), BN);
        if (cu != BN) {
#pragma unroll
          for (int c = 0; c < BN; ++c) v[c] = (c < cu || (c >= c_lo && c < c_hi)) ? v[c] : -INFINITY;
        }
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < BN; ++c) m4[c & 3] = fmaxf(m4[c & 3], v[c]);
        const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * a.scale_log2;
        if (threadIdx.x % 128 == 0) PP_TR(6, n_all);
        float alpha = 1.f;
        if (mx > m_ref + kRescale) {
          alpha = m_ref == -INFINITY ? 0.f : ex2(m_ref - mx);
          m_ref = mx;
        }
        const float nmref = m_ref == -INFINITY ? 0.f : -m_ref;
        float r4[4] = {0.f, 0.f, 0.f, 0.f};
        // P = 2^(s scale - m) as bf16 pairs over the first BN/2 columns of the S buffer
#pragma unroll
        for (int h = 0; h < BN / 32; ++h) {
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const float e0 = ex2(fmaf(v[32 * h + 2 * c], a.scale_log2, nmref));
            const float e1 = ex2(fmaf(v[32 * h + 2 * c + 1], a.scale_log2, nmref));
            r4[(2 * c) & 3] += e0;
            r4[(2 * c + 1) & 3] += e1;
            pk[c] = pack2(e0, e1);
          }
          tmem_st16(s_col + 16 * h, pk);
        }
        l_run = l_run * alpha + ((r4[0] + r4[1]) + (r4[2] + r4[3]));
        if (threadIdx.x % 128 == 0) PP_TR(7, n_all);
        if (u != 2 * P.lo) {  // PV(u-1) must have completed before O is rescaled
          mbar_wait(o_done, (n_all - 1) & 1);
          tc_after();
          if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
              float o[32];
              tmem_ld32(o_col + c * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] *= alpha;
              tmem_st32(o_col + c * 32, o);
            }
          }
        }
        tmem_wait_st();
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        if (threadIdx.x % 128 == 0) PP_TR(4, n_all);
      }
      if (threadIdx.x % 128 == 0) PP_TR(5, 3 + 2 * (pc - pb));
      // ---- epilogue: O / l and lse (base 2) into slot `part` (chunked layout:
      // a warp's 16-B stores of one 4-column chunk cover 32 consecutive rows) ----
      mbar_wait(o_done, (n_all - 1) & 1);
      tc_after();
      const uint32_t qi = q0 + r;
      const bool valid = qi < q_end;
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      float* dst = a.part_o + part_index(P.part, BM, r, 0, D);
      constexpr size_t chunk_stride = size_t(BM) * 4;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        tmem_ld32(o_col + c * 32, o);
        tmem_wait_ld();
        if (valid) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<float4*>(dst + (c * 8 + k) * chunk_stride) =
                make_float4(o[4 * k] * inv, o[4 * k + 1] * inv, o[4 * k + 2] * inv, o[4 * k + 3] * inv);
        }
      }
      if (valid) a.part_lse[size_t(P.part) * BM + r] = l_run > 0.f ? m_ref + log2f(l_run) : -INFINITY;
      if (threadIdx.x % 128 == 0) PP_TR(5, 4 + 2 * (pc - pb));
      // O is overwritten by the next piece's first PV, issued after this lane's
      // next p_full (signalled after these loads)
      tc_before();
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (threadIdx.x == 0) PP_TR(5, 2);
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
}

bool attn_pp_supported(const PoolGeom& g) {
  return (g.D == 64 || g.D == 128) && g.S >= 8 && g.S <= pp::BN && (pp::BN % g.S) == 0;  // <= 8 pages per sub-tile
}

template <int D, bool TR>
static void launch_pp(const CUtensorMap& pool_map, const CUtensorMap& q_map, const AttnArgs& a, cudaStream_t s) {
  static DeviceOnce once;
  if (once.first())
    cudaFuncSetAttribute(attn_pp_kernel<D, TR>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pp::Cfg<D>::SMEM));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.n_items / 2);  // n_items = virtual CTAs (even)
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = pp::Cfg<D>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, attn_pp_kernel<D, TR>, pool_map, q_map, a);
}

void launch_attention_pp(const CUtensorMap& pool_map, const CUtensorMap& q_map, const AttnArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return;
  if (a.g.D == 64) a.trace ? launch_pp<64, true>(pool_map, q_map, a, s) : launch_pp<64, false>(pool_map, q_map, a, s);
  else a.trace ? launch_pp<128, true>(pool_map, q_map, a, s) : launch_pp<128, false>(pool_map, q_map, a, s);
}

// Default: the column-split kernel (attn_tc.cu). Measured against this two-lane
// form on the bench layer (tools/attn_bench.py, L2 evicted): 79.4 vs 86.4 us, and
// 18.0 K vs 17.4 K requests/s on the adaptive configs[1] bench — each lane's
// 5 ring stages (its Q takes 32 KB) cover less of the ~2-3 us loaded latency
// than one pipeline's (traces: P ready -> PV issued 0.9 us, waiting for V and
// for K of S(u+2)). MTKV_ATTN=pp selects it, MTKV_ATTN=mma the mma.sync kernel.
AttnKind attn_kind(const PoolGeom& g) {
  static const int force = [] {
    const char* e = std::getenv("MTKV_ATTN");
    if (!e) return 0;
    const std::string v(e);
    return v == "mma" ? 1 : v == "pp" ? 3 : 0;
  }();
  if (force == 1 || !attn_tc_supported(g)) return AttnKind::Mma;
  if (force == 3 && attn_pp_supported(g)) return AttnKind::Pp;
  return AttnKind::Tc;
}

uint32_t attn_plan_ctas(AttnKind k, int n_sm) {
  return k == AttnKind::Pp ? 2u * uint32_t(n_sm) : k == AttnKind::Tc ? uint32_t(n_sm) : 0u;
}

void launch_attention_any(AttnKind k, const CUtensorMap& pool_map, const CUtensorMap& q_map, const AttnArgs& a,
                          cudaStream_t s) {
  if (k == AttnKind::Pp) launch_attention_pp(pool_map, q_map, a, s);
  else if (k == AttnKind::Tc && a.pair) launch_attention_pair(pool_map, q_map, a, s);
  else if (k == AttnKind::Tc) launch_attention_tc(pool_map, q_map, a, s);
  else launch_attention(a, s);
}

}  // namespace mtkv_b200
