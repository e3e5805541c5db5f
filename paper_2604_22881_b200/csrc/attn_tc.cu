// Incremental prefix-reuse attention on the 5th-gen tensor cores (sm_100a).
//
// One CTA = (request, head, 128-row query tile, key split). Warp roles:
//   warp 0      TMA producer: page-granular cp.async.bulk.tensor loads of K and V
//               straight out of the paged pool (no gather pass), 2-stage ring
//   warp 1      MMA issuer (one elected thread): S = Q K^T and O += P V with
//               tcgen05.mma kind::f16, accumulators in TMEM
//   warp 2      TMEM allocator (512 columns: S double buffer + O)
//   warps 4..7  softmax warpgroup: thread r owns query row r; tcgen05.ld of its
//               S row, mask, online softmax (base 2), P -> smem (bf16, SW128),
//               conditional O rescale in TMEM, epilogue O/l + lse to HBM
// Logical key space: the user's keys [0, KA) padded to a page boundary, then
// the request's candidate keys (their own scratch pages), so every page-sized
// slice of a tile is one TMA box. Keys past the end load as zeros (TMA OOB).
//
// Operand layouts (canonical UMMA, 128-byte swizzle, 1024-B aligned):
//   Q, P, K : K-major  [rows][64-elem blocks], SBO = 1024 B, +32 B per K=16 step
//   V       : MN-major [keys][64-dim blocks],  SBO = 1024 B, LBO = 16 KB
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>

#include "kernels.cuh"

namespace mtkv_b200 {

namespace tc {

constexpr int BM = 128;   // query rows per tile (TMEM lanes)
constexpr int BN = 64;    // keys per tile
constexpr int STAGES = 4; // K+V ring depth

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(s32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_ready(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(s32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          s32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(s32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SW128 K-major / MN-major smem descriptor (sm_100: version 1, layout 2 = SWIZZLE_128B)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo_bytes >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// byte offset of 16-byte chunk `c` (of 8) in row `r` of a SW128 K-major block
__device__ __forceinline__ uint32_t sw128(uint32_t r, uint32_t c) { return r * 128u + ((c ^ (r & 7u)) << 4); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define ATTN_TR(kind, t)                                                                  \
  do {                                                                                    \
    if (a.trace && blockIdx.x < kTraceCtas && (t) < kTraceTiles)                          \
      a.trace[((size_t)blockIdx.x * kTraceKinds + (kind)) * kTraceTiles + (t)] = gtime(); \
  } while (0)

struct Smem {
  static constexpr uint32_t kBlock = BM * 128;  // one 128-row x 64-elem bf16 block = 16 KB
};

}  // namespace tc

using namespace tc;

// Two softmax pipelines per CTA: warpgroup p in {0,1} owns key tiles t with
// t % 2 == p, its own S and O accumulators in TMEM and its own P buffer, and
// writes its result as partial (2*split + p); the split-K merge in
// gate_norm_kernel combines them. While one warpgroup runs softmax the tensor
// core works on the other pipeline's S / PV, so neither unit waits on the other.
template <int D>
__global__ void __launch_bounds__(384, 1) attn_tc_kernel(const __grid_constant__ CUtensorMap pool_map, AttnArgs a) {
  constexpr int NB = D / 64;                            // 64-element column blocks of Q/K/V
  constexpr uint32_t QBLK = BM * 128;                   // Q/P block: 128 rows x 128 B
  constexpr uint32_t KBLK = BN * 128;                   // K/V block: BN rows x 128 B
  constexpr uint32_t Q_BYTES = NB * QBLK;
  constexpr uint32_t P_BYTES = (BN / 64) * QBLK;        // 128 rows x BN keys (per pipeline)
  constexpr uint32_t KV_BYTES = NB * KBLK;              // BN keys x D (K or V)
  constexpr uint32_t STAGE_BYTES = 2 * KV_BYTES;
  constexpr uint32_t PIPE_COLS = BN + D;                // S + O per pipeline
  constexpr uint32_t TMEM_COLS = 2 * PIPE_COLS <= 256 ? 256 : 512;
  constexpr float kRescale = 8.f;                       // lazy rescale threshold (log2 units)

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sP = sQ + Q_BYTES;                 // [2] pipelines
  uint8_t* sKV = sP + 2 * P_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + STAGES * STAGE_BYTES);
  uint64_t* full = bars;                 // [STAGES] K+V of a tile landed
  uint64_t* empty = bars + STAGES;       // [STAGES] stage consumed by PV
  uint64_t* s_full = bars + 2 * STAGES;  // [2 pipes] S tile in TMEM
  uint64_t* s_free = s_full + 2;         // [2] S read by softmax
  uint64_t* p_full = s_free + 2;         // [2] P in smem (+ O rescaled)
  uint64_t* o_done = p_full + 2;         // [2] PV committed
  uint64_t* q_full = o_done + 2;         // Q in smem
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 1);

  const AttnItem it = a.items[blockIdx.x];
  const ReqDev R = a.reqs[it.req];
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const PoolGeom& g = a.g;
  const uint32_t S = g.S, h = it.head;
  if (threadIdx.x == 0) ATTN_TR(5, 0);

  // logical key space: user keys [0, KA) padded to KAp, then candidates
  const uint64_t KA = R.start + R.n_hist;
  const uint64_t KAp = (KA + S - 1) / S * S;
  const uint32_t user_pages = uint32_t(KAp / S);
  const uint32_t q0 = it.qtile * BM;
  const uint32_t q_end = min(R.n_q, q0 + BM);
  const uint64_t pos_last = R.start + q_end - 1;
  const uint64_t k_vis = pos_last >= KA ? KAp + (pos_last - KA + 1) : pos_last + 1;
  const uint64_t k_lo = uint64_t(it.split) * R.split_keys;
  const uint64_t k_hi = min(k_vis, k_lo + uint64_t(R.split_keys));
  const int n_tiles = k_hi > k_lo ? int((k_hi - k_lo + BN - 1) / BN) : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int p = 0; p < 2; ++p) {
      mbar_init(&s_full[p], 1);
      mbar_init(&s_free[p], 4);
      mbar_init(&p_full[p], 4);
      mbar_init(&o_done[p], 1);
    }
    mbar_init(q_full, 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) ATTN_TR(5, 1);

  if (warp == 0) {
    // ---------------- TMA producer (whole warp: lane i resolves page i) ----------------
    if (n_tiles > 0) {
      const int ppt = BN / S;  // pages per tile
      auto row_of = [&](uint64_t lp) -> int {  // pool row of a logical page's K slice
        if (lp < user_pages) {
          const uint32_t page = a.pages[R.pages_off + uint32_t(lp)];
          return int(((uint64_t(a.layer) * g.num_pages + page) * 2) * S);
        }
        if (lp - user_pages < R.n_scratch && (lp - user_pages) * S < R.n_cand) {
          const uint32_t page = a.pages[R.scratch_off + uint32_t(lp - user_pages)];
          return int(((uint64_t(a.layer) * g.num_pages + page) * 2) * S);
        }
        return -int(S) * 4;  // out of bounds -> TMA zero fill
      };
      const uint64_t lp_base = k_lo / S;
      int rows_cache = row_of(lp_base + lane);  // 32 consecutive pages per refresh
      int cache_tile0 = 0;
      for (int t = 0; t < n_tiles; ++t) {
        const int st = t % STAGES;
        if ((t - cache_tile0) * ppt >= 32) {
          cache_tile0 = t;
          rows_cache = row_of(lp_base + uint64_t(t) * ppt + lane);
        }
        if (lane == 0) {
          if (t >= STAGES) mbar_wait(&empty[st], ((t / STAGES) - 1) & 1);
          ATTN_TR(0, t);
          mbar_expect_tx(&full[st], STAGE_BYTES);
        }
        __syncwarp();
        uint8_t* kdst = sKV + st * STAGE_BYTES;
        uint8_t* vdst = kdst + KV_BYTES;
        for (int i = 0; i < ppt; ++i) {
          const int row_k = __shfl_sync(0xffffffffu, rows_cache, (t - cache_tile0) * ppt + i);
          const int row_v = row_k >= 0 ? row_k + int(S) : row_k;
          if (lane == 0) {
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              tma_load_2d(kdst + b * KBLK + i * S * 128, &pool_map, int(h * D + 64 * b), row_k, &full[st]);
              tma_load_2d(vdst + b * KBLK + i * S * 128, &pool_map, int(h * D + 64 * b), row_v, &full[st]);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: non-blocking event loop over both pipelines ----------------
    if (lane == 0 && n_tiles > 0) {
      constexpr uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
      constexpr uint32_t idesc_o =
          (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(D >> 3) << 17) | (uint32_t(BM >> 4) << 24);
      const uint32_t q_addr = s32(sQ);
      mbar_wait(q_full, 0);
      tc_after();
      int next_s = 0, next_pv = 0;
      while (next_pv < n_tiles) {
        bool progressed = false;
        // PV first: it frees a K/V stage and unblocks the owning softmax warpgroup
        if (next_pv < next_s) {
          const int t = next_pv, p = t & 1, u = t >> 1, st = t % STAGES;
          if (mbar_ready(&p_full[p], u & 1)) {
            tc_after();
            const uint32_t p_addr = s32(sP + p * P_BYTES);
            const uint32_t v_addr = s32(sKV + st * STAGE_BYTES + KV_BYTES);
#pragma unroll
            for (int k = 0; k < BN / 16; ++k) {
              const uint64_t pa = sdesc(p_addr + (k / 4) * QBLK + (k % 4) * 32, 16, 1024);
              const uint64_t vb = sdesc(v_addr + k * 2048, KBLK, 1024);  // MN-major V, LBO = KBLK
              mma_f16(tmem + p * PIPE_COLS + BN, pa, vb, idesc_o, (u > 0 || k > 0) ? 1u : 0u);
            }
            mma_commit(&o_done[p]);
            mma_commit(&empty[st]);
            ATTN_TR(2, t);
            ++next_pv;
            progressed = true;
          }
        }
        if (next_s < n_tiles && next_s < next_pv + 2) {  // at most one S ahead per pipeline
          const int t = next_s, p = t & 1, u = t >> 1, st = t % STAGES;
          if (mbar_ready(&full[st], (t / STAGES) & 1) && (u == 0 || mbar_ready(&s_free[p], (u - 1) & 1))) {
            tc_after();
            const uint32_t k_addr = s32(sKV + st * STAGE_BYTES);
#pragma unroll
            for (int k = 0; k < D / 16; ++k)
              mma_f16(tmem + p * PIPE_COLS, sdesc(q_addr + (k / 4) * QBLK + (k % 4) * 32, 16, 1024),
                      sdesc(k_addr + (k / 4) * KBLK + (k % 4) * 32, 16, 1024), idesc_s, k > 0);
            mma_commit(&s_full[p]);
            ATTN_TR(1, t);
            ++next_s;
            progressed = true;
          }
        }
        if (!progressed) __nanosleep(20);
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax warpgroups ----------------
    const uint32_t p = (warp - 4) / 4;          // pipeline
    const uint32_t r = (threadIdx.x - 128) % 128;  // query row == TMEM lane
    const uint32_t lane_base = (32u * (warp % 4)) << 16;
    const uint32_t s_col = p * PIPE_COLS, o_col = p * PIPE_COLS + BN;
    uint8_t* myP = sP + p * P_BYTES;
    // Q row -> smem (SW128 K-major); each warpgroup writes half of the row's blocks
    {
      const uint32_t qi = q0 + r;
      const bool ok = qi < R.n_q;
      const uint4* src = reinterpret_cast<const uint4*>(a.q + size_t(R.q_row0 + (ok ? qi : 0)) * g.d + h * D);
#pragma unroll
      for (int c = p; c < D / 8; c += 2) {
        uint4 v = ok ? src[c] : make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(sQ + (c / 8) * QBLK + sw128(r, c % 8)) = v;
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_full);
    }
    const uint64_t pos_r = R.start + q0 + r;
    // valid keys of this row: user keys [0, u_end), candidate keys [KAp, c_end)
    const uint64_t u_end = min(min(KA, k_hi), pos_r + 1);
    const uint64_t c_end = pos_r >= KA ? min(min(KAp + R.n_cand, KAp + (pos_r - KA + 1)), k_hi) : KAp;
    float m_ref = -INFINITY, l_run = 0.f;
    int u = 0;
    for (int t = p; t < n_tiles; t += 2, ++u) {
      mbar_wait(&s_full[p], u & 1);
      tc_after();
      if (threadIdx.x % 128 == 0) ATTN_TR(3, t);
      float s[BN];
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) tmem_ld32(tmem + lane_base + s_col + c * 32, s + c * 32);
      tmem_wait_ld();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[p]);
      const uint64_t kb = k_lo + uint64_t(t) * BN;
      const int cu = int(u_end > kb ? (u_end - kb < uint64_t(BN) ? u_end - kb : uint64_t(BN)) : 0);
      const int c_lo = int(KAp > kb ? (KAp - kb < uint64_t(BN) ? KAp - kb : uint64_t(BN)) : 0);
      const int c_hi = int(c_end > kb ? (c_end - kb < uint64_t(BN) ? c_end - kb : uint64_t(BN)) : 0);
      float mx = -INFINITY;
      if (cu == BN) {
#pragma unroll
        for (int c = 0; c < BN; ++c) {
          s[c] *= a.scale_log2;
          mx = fmaxf(mx, s[c]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < BN; ++c) {
          const bool ok = c < cu || (c >= c_lo && c < c_hi);
          s[c] = ok ? s[c] * a.scale_log2 : -INFINITY;
          mx = fmaxf(mx, s[c]);
        }
      }
      float alpha = 1.f;
      if (mx > m_ref + kRescale) {  // lazy rescale: p <= 2^8 between rescales
        alpha = m_ref == -INFINITY ? 0.f : ex2(m_ref - mx);
        m_ref = mx;
      }
      const float mref = m_ref == -INFINITY ? 0.f : m_ref;
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < BN; ++c) {
        s[c] = ex2(s[c] - mref);
        rs += s[c];
      }
      l_run = l_run * alpha + rs;
      if (u > 0) {  // this pipeline's previous PV must finish before O / P are touched
        mbar_wait(&o_done[p], (u - 1) & 1);
        tc_after();
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            float o[32];
            tmem_ld32(tmem + lane_base + o_col + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tmem_st32(tmem + lane_base + o_col + c * 32, o);
          }
          tmem_wait_st();
        }
      }
#pragma unroll
      for (int c = 0; c < BN / 8; ++c) {
        uint4 v;
        v.x = pack2(s[c * 8 + 0], s[c * 8 + 1]);
        v.y = pack2(s[c * 8 + 2], s[c * 8 + 3]);
        v.z = pack2(s[c * 8 + 4], s[c * 8 + 5]);
        v.w = pack2(s[c * 8 + 6], s[c * 8 + 7]);
        *reinterpret_cast<uint4*>(myP + (c / 8) * QBLK + sw128(r, c % 8)) = v;
      }
      fence_async_smem();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[p]);
      if (threadIdx.x % 128 == 0) ATTN_TR(4, t);
    }
    // epilogue: this pipeline's O / l and lse (base 2) as partial 2*split + p
    const uint32_t qi = q0 + r;
    if (u > 0) {
      mbar_wait(&o_done[p], (u - 1) & 1);
      tc_after();
    }
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
    const size_t prow = size_t(R.part_base) + (size_t(it.split) * 2 + p) * R.n_q + qi;
    float* dst = a.part_o + prow * g.d + h * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float o[32];
      if (u > 0) {
        tmem_ld32(tmem + lane_base + o_col + c * 32, o);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = 0.f;
      }
      if (qi < q_end) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(dst + c * 32 + i) = make_float4(o[i] * inv, o[i + 1] * inv, o[i + 2] * inv, o[i + 3] * inv);
      }
    }
    if (qi < q_end) a.part_lse[prow * g.H + h] = l_run > 0.f ? m_ref + log2f(l_run) : -INFINITY;
    if (threadIdx.x == 128) ATTN_TR(5, 2);
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
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

bool attn_tc_supported(const PoolGeom& g) {
  return (g.D == 64 || g.D == 128) && g.S >= 8 && g.S <= 128 && (128 % g.S) == 0;
}

int make_pool_map(CUtensorMap* map, const void* pool, const PoolGeom& g) {
  const cuuint64_t rows = cuuint64_t(g.L) * g.num_pages * 2 * g.S;
  const cuuint64_t dims[2] = {g.d, rows};
  const cuuint64_t strides[1] = {cuuint64_t(g.d) * 2};
  const cuuint32_t box[2] = {64, g.S};
  const cuuint32_t estr[2] = {1, 1};
  auto fn = encode_fn();
  if (!fn) return -1;
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

template <int D>
static void launch_tc_d(const CUtensorMap& map, const AttnArgs& a, cudaStream_t s) {
  constexpr size_t smem = 1024 + (D / 64) * BM * 128 + 2 * (BN / 64) * BM * 128 + STAGES * 2 * (D / 64) * BN * 128 + 256;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(attn_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    set = true;
  }
  attn_tc_kernel<D><<<a.n_items, 384, smem, s>>>(map, a);
}

void launch_attention_tc(const CUtensorMap& map, const AttnArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return;
  if (a.g.D == 64) launch_tc_d<64>(map, a, s);
  else launch_tc_d<128>(map, a, s);
}

}  // namespace mtkv_b200
