// CUDA kernels of the serving path (sm_100a). See kernels.cuh for layouts.
//
//   gemm_kernel        bf16 x bf16 -> fp32 tensor-core GEMM with fused epilogues;
//                      the Proj epilogue is Alg. 1 step 8.1 + 8.2: silu(e W_in),
//                      split u|q|k|v, and append k,v straight into the paged pool
//                      (reference: model.cpp:146-160 + store.hpp:123 append).
//   attn_kernel        incremental prefix-reuse attention over paged K/V,
//                      split-K over key ranges (model.cpp:104 attention).
//   gate_norm_kernel   split combine, silu(o)*u, layer norm (model.cpp:164-165).
//   scatter/gather     onload-buffer <-> pages, 128-bit vector copies
//                      (store.hpp:89 scatter / :106 gather).
//   tag_append_kernel  tag backend payload (store.hpp:19).
#include "kernels.cuh"

#include <cfloat>
#include <cstdlib>
#include <cmath>

namespace mtkv_b200 {

// ------------------------------------------------------------- primitives ---
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;  // zero-fill when invalid
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void ldsm_x4(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float silu_f(float x) { return __fdividef(x, 1.0f + __expf(-x)); }

// ------------------------------------------------------------------- GEMM ---
// 64x64x32 block tile, 4 warps (2x2, 32x32 each), double-buffered smem.
// VEC: 16-byte cp.async loads (K % 8 == 0, N % 8 == 0); otherwise scalar loads.
constexpr int GBM = 64, GBN = 64, GBK = 32, GLA = GBK + 8, GLB = GBN + 8;

template <bool VEC>
__device__ __forceinline__ void gemm_load_tile(const GemmArgs& a, __nv_bfloat16 (*As)[GLA],
                                               __nv_bfloat16 (*Bs)[GLB], int m0, int n0, int k0,
                                               int tid) {
  if constexpr (VEC) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int c = tid + i * 128, row = c >> 2, kc = (c & 3) * 8;
      const int m = m0 + row, k = k0 + kc;
      const bool ok = m < a.M && k < a.K;
      const int src_row = ok ? (a.row_idx ? (int)a.row_idx[m] : m) : 0;
      cp_async16(&As[row][kc], a.A + (size_t)src_row * a.K + (ok ? k : 0), ok);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int c = tid + i * 128, row = c >> 3, nc = (c & 7) * 8;
      const int k = k0 + row, n = n0 + nc;
      const bool ok = k < a.K && n < a.N;
      cp_async16(&Bs[row][nc], a.B + (ok ? (size_t)k * a.N + n : 0), ok);
    }
  } else {
    for (int c = tid; c < GBM * GBK; c += 128) {
      const int row = c / GBK, kc = c % GBK, m = m0 + row, k = k0 + kc;
      __nv_bfloat16 v = __float2bfloat16(0.f);
      if (m < a.M && k < a.K) v = a.A[(size_t)(a.row_idx ? (int)a.row_idx[m] : m) * a.K + k];
      As[row][kc] = v;
    }
    for (int c = tid; c < GBK * GBN; c += 128) {
      const int row = c / GBN, nc = c % GBN, k = k0 + row, n = n0 + nc;
      __nv_bfloat16 v = __float2bfloat16(0.f);
      if (k < a.K && n < a.N) v = a.B[(size_t)k * a.N + n];
      Bs[row][nc] = v;
    }
  }
}

template <bool VEC>
__global__ void __launch_bounds__(128) gemm_kernel(GemmArgs a) {
  __shared__ __align__(16) __nv_bfloat16 As[2][GBM][GLA];
  __shared__ __align__(16) __nv_bfloat16 Bs[2][GBK][GLB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  float acc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.f;

  const int nk = (a.K + GBK - 1) / GBK;
  gemm_load_tile<VEC>(a, As[0], Bs[0], m0, n0, 0, tid);
  cp_commit();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) {
      gemm_load_tile<VEC>(a, As[buf ^ 1], Bs[buf ^ 1], m0, n0, (kt + 1) * GBK, tid);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK / 16; ++kk) {
      uint32_t af[2][4], bf[2][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
        ldsm_x4(af[mt], &As[buf][wm * 32 + mt * 16 + (lane & 15)][kk * 16 + (lane >> 4) * 8]);
#pragma unroll
      for (int np = 0; np < 2; ++np)
        ldsm_x4_t(bf[np], &Bs[buf][kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8][wn * 32 + np * 16 + (lane >> 4) * 8]);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          mma16816(acc[mt][nt], af[mt], bf[nt >> 1][(nt & 1) * 2], bf[nt >> 1][(nt & 1) * 2 + 1]);
    }
    __syncthreads();
  }

  // epilogue
  const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int row = m0 + wm * 32 + mt * 16 + gq + hr * 8;
      if (row >= a.M) continue;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int col = n0 + wn * 32 + nt * 8 + tq * 2;
        if (col >= a.N) continue;
        float v0 = acc[mt][nt][hr * 2], v1 = acc[mt][nt][hr * 2 + 1];
        const bool two = col + 1 < a.N;
        switch (a.epi) {
          case Epi::F32: {
            float* o = static_cast<float*>(a.out) + (size_t)row * a.N + col;
            o[0] = v0;
            if (two) o[1] = v1;
            break;
          }
          case Epi::Bf16:
          case Epi::SiluBf16: {
            if (a.epi == Epi::SiluBf16) { v0 = silu_f(v0); v1 = silu_f(v1); }
            __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out) + (size_t)row * a.N + col;
            if (two && ((((size_t)row * a.N + col) & 1) == 0)) {
              *reinterpret_cast<__nv_bfloat162*>(o) = __floats2bfloat162_rn(v0, v1);
            } else {
              o[0] = __float2bfloat16(v0);
              if (two) o[1] = __float2bfloat16(v1);
            }
            break;
          }
          case Epi::Proj: {
            v0 = silu_f(v0);
            v1 = silu_f(v1);
            const uint32_t part = col / a.d, w = col % a.d;  // d even: pair stays in one part
            __nv_bfloat16* dst;
            if (part == 0) dst = a.out_u + (size_t)row * a.d + w;
            else if (part == 1) dst = a.out_q + (size_t)row * a.d + w;
            else dst = a.pool + a.layer_base + a.kv_off[row] + (part == 3 ? a.kv_stride : 0) + w;
            *reinterpret_cast<__nv_bfloat162*>(dst) = __floats2bfloat162_rn(v0, v1);
            break;
          }
        }
      }
    }
}

void launch_gemm(const GemmArgs& a, cudaStream_t s) {
  if (a.M <= 0) return;
  dim3 grid((a.N + GBN - 1) / GBN, (a.M + GBM - 1) / GBM);
  const bool vec = (a.K % 8 == 0) && (a.N % 8 == 0);
  if (vec) gemm_kernel<true><<<grid, 128, 0, s>>>(a);
  else gemm_kernel<false><<<grid, 128, 0, s>>>(a);
}

// one warp per row: 16-B vector copies of the token's embedding row when d % 8 == 0
__global__ void embed_kernel(__nv_bfloat16* x, const __nv_bfloat16* table, const uint32_t* tok, int rows, int d) {
  const int r = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (r >= rows) return;
  const __nv_bfloat16* src = table + (size_t)tok[r] * d;
  __nv_bfloat16* dst = x + (size_t)r * d;
  if (d % 8 == 0) {
    for (int j = lane * 8; j < d; j += 32 * 8)
      *reinterpret_cast<uint4*>(dst + j) = *reinterpret_cast<const uint4*>(src + j);
  } else {
    for (int j = lane; j < d; j += 32) dst[j] = src[j];
  }
}

void launch_embed(__nv_bfloat16* x, const __nv_bfloat16* table, const uint32_t* tok, int rows, int d,
                  cudaStream_t s) {
  if (rows > 0) embed_kernel<<<(rows + 7) / 8, 256, 0, s>>>(x, table, tok, rows, d);
}

// -------------------------------------------------------------- attention ---
// One CTA = (request, head, 64-query tile, key split). 4 warps x 16 query rows.
// Keys stream page by page through a 2-stage cp.async ring (64 keys/stage).
// Key index == position: indices [0, start+n_hist) live in the user's pages,
// [start+n_hist, start+n_hist+n_cand) in the request's scratch pages.
constexpr int ABK = 64;

__device__ __forceinline__ const __nv_bfloat16* key_row(const AttnArgs& a, const ReqDev& R, uint64_t idx,
                                                        uint32_t kv, uint32_t h) {
  const uint64_t KA = R.start + R.n_hist;
  uint32_t page, slot;
  if (idx < KA) {
    page = a.pages[R.pages_off + (uint32_t)(idx / a.g.S)];
    slot = (uint32_t)(idx % a.g.S);
  } else {
    const uint64_t c = idx - KA;
    page = a.pages[R.scratch_off + (uint32_t)(c / a.g.S)];
    slot = (uint32_t)(c % a.g.S);
  }
  return a.pool + a.g.off(a.layer, page, kv, slot) + (size_t)h * a.g.D;
}

template <int DP, bool VEC, int NT>
__device__ __forceinline__ void attn_load_kv(const AttnArgs& a, const ReqDev& R, __nv_bfloat16* Ks,
                                             __nv_bfloat16* Vs, uint64_t k0, uint64_t k_hi, uint32_t h,
                                             int tid) {
  constexpr int LD = DP + 8, CH = DP / 8;
  const uint32_t D = a.g.D;
  if constexpr (VEC) {
    const int live = (int)((D + 7) / 8);
    for (int c = tid; c < ABK * CH; c += NT) {
      const int row = c / CH, ch = c % CH;
      if (ch >= live) continue;
      const uint64_t idx = k0 + row;
      const bool ok = idx < k_hi;
      const __nv_bfloat16* kr = ok ? key_row(a, R, idx, 0, h) : a.pool;
      const __nv_bfloat16* vr = ok ? kr + (size_t)a.g.S * a.g.d : a.pool;
      cp_async16(Ks + row * LD + ch * 8, kr + (ok ? ch * 8 : 0), ok);
      cp_async16(Vs + row * LD + ch * 8, vr + (ok ? ch * 8 : 0), ok);
    }
  } else {
    for (int c = tid; c < ABK * (int)D; c += NT) {
      const int row = c / D, j = c % D;
      const uint64_t idx = k0 + row;
      __nv_bfloat16 kv0 = __float2bfloat16(0.f), kv1 = __float2bfloat16(0.f);
      if (idx < k_hi) {
        const __nv_bfloat16* kr = key_row(a, R, idx, 0, h);
        kv0 = kr[j];
        kv1 = kr[(size_t)a.g.S * a.g.d + j];
      }
      Ks[row * LD + j] = kv0;
      Vs[row * LD + j] = kv1;
    }
  }
}

// NW warps x 16 query rows = one query tile; K/V of the split are streamed once
// per tile, so a request whose fresh rows fit one tile reads its prefix once.
template <int DP, bool VEC, int NW>
__global__ void __launch_bounds__(NW * 32) attn_kernel(AttnArgs a) {
  constexpr int LD = DP + 8, NKT = ABK / 8, NDT = DP / 8, NT = NW * 32, ABQ = NW * 16;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* Kb = Qs + ABQ * LD;
  __nv_bfloat16* Vb = Kb + 2 * ABK * LD;

  const AttnItem it = a.items[blockIdx.x];
  const ReqDev R = a.reqs[it.req];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const uint32_t D = a.g.D, d = a.g.d, h = it.head;
  const uint64_t n_keys = R.start + R.n_hist + R.n_cand;
  const uint32_t q0 = it.qtile * ABQ;
  const uint32_t q_end = min(R.n_q, q0 + ABQ);
  const uint64_t k_vis = min(n_keys, R.start + q_end);
  const uint64_t k_lo = (uint64_t)it.split * R.split_keys;
  const uint64_t k_hi = min(k_vis, k_lo + (uint64_t)R.split_keys);

  // zero everything once: pad columns and masked rows stay finite
  for (int i = tid; i < (ABQ + 4 * ABK) * LD / 8; i += NT)
    reinterpret_cast<uint4*>(smem_raw)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  // Q tile
  for (int c = tid; c < ABQ * (int)D; c += NT) {
    const int row = c / D, j = c % D;
    if (q0 + row < q_end) Qs[row * LD + j] = a.q[(size_t)(R.q_row0 + q0 + row) * d + h * D + j];
  }
  const int n_tiles = k_hi > k_lo ? (int)((k_hi - k_lo + ABK - 1) / ABK) : 0;
  if (n_tiles > 0) {
    attn_load_kv<DP, VEC, NT>(a, R, Kb, Vb, k_lo, k_hi, h, tid);
    cp_commit();
  }
  __syncthreads();

  uint32_t qf[DP / 16][4];
#pragma unroll
  for (int kk = 0; kk < DP / 16; ++kk)
    ldsm_x4(qf[kk], Qs + (warp * 16 + (lane & 15)) * LD + kk * 16 + (lane >> 4) * 8);

  const uint64_t pos_r0 = R.start + q0 + warp * 16 + gq, pos_r1 = pos_r0 + 8;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  float o[NDT][4];
#pragma unroll
  for (int i = 0; i < NDT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;

  for (int t = 0; t < n_tiles; ++t) {
    const int buf = t & 1;
    const uint64_t kbase = k_lo + (uint64_t)t * ABK;
    if (t + 1 < n_tiles) {
      attn_load_kv<DP, VEC, NT>(a, R, Kb + (buf ^ 1) * ABK * LD, Vb + (buf ^ 1) * ABK * LD, kbase + ABK, k_hi, h, tid);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const __nv_bfloat16* Ks = Kb + buf * ABK * LD;
    const __nv_bfloat16* Vs = Vb + buf * ABK * LD;

    float s[NKT][4];
#pragma unroll
    for (int i = 0; i < NKT; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DP / 16; ++kk)
#pragma unroll
      for (int np = 0; np < NKT / 2; ++np) {
        uint32_t b[4];
        ldsm_x4(b, Ks + (np * 16 + (lane & 7) + (lane >> 4) * 8) * LD + kk * 16 + ((lane >> 3) & 1) * 8);
        mma16816(s[2 * np], qf[kk], b[0], b[1]);
        mma16816(s[2 * np + 1], qf[kk], b[2], b[3]);
      }

    // mask + online softmax (base-2)
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < NKT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint64_t key = kbase + nt * 8 + tq * 2 + (e & 1);
        const uint64_t pos = (e < 2) ? pos_r0 : pos_r1;
        const bool ok = key < k_hi && key <= pos;
        s[nt][e] = ok ? s[nt][e] * a.scale_log2 : -INFINITY;
        mx[e >> 1] = fmaxf(mx[e >> 1], s[nt][e]);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 2));
    }
    float alpha[2], mref[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float mn = fmaxf(m_r[r], mx[r]);
      mref[r] = (mn == -INFINITY) ? 0.f : mn;
      alpha[r] = (m_r[r] == -INFINITY) ? 0.f : exp2f(m_r[r] - mref[r]);
      m_r[r] = mn;
    }
    float rs[2] = {0.f, 0.f};
#pragma unroll
    for (int nt = 0; nt < NKT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = exp2f(s[nt][e] - mref[e >> 1]);  // -inf -> 0
        s[nt][e] = p;
        rs[e >> 1] += p;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) l_r[r] = l_r[r] * alpha[r] + rs[r];
#pragma unroll
    for (int i = 0; i < NDT; ++i) {
      o[i][0] *= alpha[0]; o[i][1] *= alpha[0];
      o[i][2] *= alpha[1]; o[i][3] *= alpha[1];
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < ABK / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int np = 0; np < NDT / 2; ++np) {
        uint32_t b[4];
        ldsm_x4_t(b, Vs + (kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LD + np * 16 + (lane >> 4) * 8);
        mma16816(o[2 * np], pa, b[0], b[1]);
        mma16816(o[2 * np + 1], pa, b[2], b[3]);
      }
    }
    __syncthreads();
  }

  // finalize partial: O / l and lse (base 2)
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffff, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffff, l_r[r], 2);
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const uint32_t qi = q0 + warp * 16 + gq + r * 8;
    if (qi >= q_end) continue;
    const AttnSeg& sg = a.segs[R.seg0 + h * R.qtiles + it.qtile];
    const uint32_t slot = sg.part_base + it.split;
    const size_t prow = (size_t)slot * ABQ + (qi - q0);
    const float inv = l_r[r] > 0.f ? 1.f / l_r[r] : 0.f;
#pragma unroll
    for (int i = 0; i < NDT; ++i) {
      const uint32_t col = i * 8 + tq * 2;
      if (col < D) a.part_o[part_index(slot, ABQ, qi - q0, col, D)] = o[i][r * 2] * inv;
      if (col + 1 < D) a.part_o[part_index(slot, ABQ, qi - q0, col + 1, D)] = o[i][r * 2 + 1] * inv;
    }
    if (tq == 0) a.part_lse[prow] = l_r[r] > 0.f ? m_r[r] + log2f(l_r[r]) : -INFINITY;
  }
}

template <int DP, bool VEC, int NW>
static void launch_attn_cfg(const AttnArgs& a, cudaStream_t s) {
  const size_t smem = (size_t)(NW * 16 + 4 * ABK) * (DP + 8) * sizeof(__nv_bfloat16);
  static DeviceOnce once;
  if (once.first()) cudaFuncSetAttribute(attn_kernel<DP, VEC, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  attn_kernel<DP, VEC, NW><<<a.n_items, NW * 32, smem, s>>>(a);
}

template <int DP>
static void launch_attn_dp(const AttnArgs& a, cudaStream_t s) {
  const bool vec = (a.g.D % 8 == 0);
  if (a.bq == 128) {
    if (vec) launch_attn_cfg<DP, true, 8>(a, s); else launch_attn_cfg<DP, false, 8>(a, s);
  } else {
    if (vec) launch_attn_cfg<DP, true, 4>(a, s); else launch_attn_cfg<DP, false, 4>(a, s);
  }
}

void launch_attention(const AttnArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return;
  if (a.g.D <= 16) launch_attn_dp<16>(a, s);
  else if (a.g.D <= 32) launch_attn_dp<32>(a, s);
  else if (a.g.D <= 64) launch_attn_dp<64>(a, s);
  else launch_attn_dp<128>(a, s);
}

// ------------------------------------------------------------- gate/norm ---
// One warp per fresh row: merge the row's partial slots per head (log-sum-exp
// weights, base 2), silu(o) * u, layer norm. When d % 32 == 0 and the head
// width is a multiple of d/32, each lane owns d/32 contiguous columns of one
// head (vector loads of every slot); otherwise lanes stride the columns.
constexpr int GATE_WARPS = 8, GATE_MAXE = 16;  // d <= 512

__device__ __forceinline__ float gate_merge_col(const GateArgs& a, const AttnSeg& sg, uint32_t ri, uint32_t c) {
  float mx = -INFINITY;
  for (uint32_t k = 0; k < sg.n_parts; ++k) mx = fmaxf(mx, a.part_lse[(size_t)(sg.part_base + k) * a.bm + ri]);
  float num = 0.f, den = 0.f;
  for (uint32_t k = 0; k < sg.n_parts; ++k) {
    const size_t prow = (size_t)(sg.part_base + k) * a.bm + ri;
    const float l = a.part_lse[prow];
    if (l == -INFINITY) continue;
    const float w = exp2f(l - mx);
    num += w * a.part_o[part_index(sg.part_base + k, a.bm, ri, c, a.D)];
    den += w;
  }
  return den > 0.f ? num / den : 0.f;
}

template <int E>  // contiguous columns per lane
__global__ void __launch_bounds__(GATE_WARPS * 32) gate_norm_kernel(GateArgs a) {
  // launched with PDL behind the attention: wait for its partials, let the MLP GEMM launch
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int wid = threadIdx.x / 32;
  const int row = blockIdx.x * GATE_WARPS + wid;
  const int lane = threadIdx.x & 31;
  if (row >= (int)a.rows) return;
  const ReqDev R = a.reqs[a.row_req[row]];
  const uint32_t i = row - R.q_row0, qt = i / a.bm, ri = i % a.bm, d = a.H * a.D;
  const size_t urow = a.u_rows ? a.u_rows[row] : uint32_t(row);  // gate operand's batch row
  constexpr int NE = E > 0 ? E : GATE_MAXE;
  float x[NE];
  float sum = 0.f;
  if constexpr (E > 0) {
    const uint32_t j0 = lane * E, h = j0 / a.D, c0 = j0 % a.D;
    // the gate operand does not depend on the merge: its load overlaps the slot reads
    float ug[E];
    {
      const __nv_bfloat16* up = a.u + urow * d + j0;
      if constexpr (E % 8 == 0) {
#pragma unroll
        for (int e = 0; e < E; e += 8) {
          const uint4 pk = *reinterpret_cast<const uint4*>(up + e);
          const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&pk);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 f = __bfloat1622float2(p2[k]);
            ug[e + 2 * k] = f.x;
            ug[e + 2 * k + 1] = f.y;
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) ug[e] = __bfloat162float(up[e]);
      }
    }
    const AttnSeg sg = a.segs[R.seg0 + h * R.qtiles + qt];
    float mx = -INFINITY;
    for (uint32_t k = 0; k < sg.n_parts; ++k) mx = fmaxf(mx, a.part_lse[(size_t)(sg.part_base + k) * a.bm + ri]);
    float acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = 0.f;
    float den = 0.f;
    for (uint32_t k = 0; k < sg.n_parts; ++k) {
      const size_t prow = (size_t)(sg.part_base + k) * a.bm + ri;
      const float l = a.part_lse[prow];
      if (l == -INFINITY) continue;
      const float w = exp2f(l - mx);
      den += w;
      if constexpr (E % 4 == 0) {  // c0 % 4 == 0: every 4 columns are one chunk of the slot
#pragma unroll
        for (int e = 0; e < E; e += 4) {
          const float4 v = *reinterpret_cast<const float4*>(a.part_o + part_index(sg.part_base + k, a.bm, ri, c0 + e, a.D));
          acc[e] += w * v.x; acc[e + 1] += w * v.y; acc[e + 2] += w * v.z; acc[e + 3] += w * v.w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] += w * a.part_o[part_index(sg.part_base + k, a.bm, ri, c0 + e, a.D)];
      }
    }
    const float inv = den > 0.f ? 1.f / den : 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const float o = acc[e] * inv;
      x[e] = silu_f(o) * ug[e];
      sum += x[e];
    }
  } else {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const uint32_t j = lane + 32 * e;
      x[e] = 0.f;
      if (j >= d) continue;
      const uint32_t h = j / a.D;
      const AttnSeg sg = a.segs[R.seg0 + h * R.qtiles + qt];
      const float o = gate_merge_col(a, sg, ri, j % a.D);
      x[e] = silu_f(o) * __bfloat162float(a.u[urow * d + j]);
      sum += x[e];
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffff, sum, off);
  const float mean = sum / (float)d;
  float var = 0.f;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const uint32_t j = E > 0 ? lane * E + e : lane + 32 * e;
    if (j < d) { const float c = x[e] - mean; var += c * c; }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) var += __shfl_xor_sync(0xffffffff, var, off);
  var /= (float)d;
  const float inv = 1.0f / sqrtf(var + 1e-6f);
  if constexpr (E > 0) {
    __nv_bfloat16* op = a.out + (size_t)row * d + lane * E;
    if constexpr (E % 8 == 0) {
#pragma unroll
      for (int e = 0; e < E; e += 8) {
        const float4 s0 = *reinterpret_cast<const float4*>(a.ln_scale + lane * E + e);
        const float4 s1 = *reinterpret_cast<const float4*>(a.ln_scale + lane * E + e + 4);
        const float sc[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
        uint4 pk;
        uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const __nv_bfloat162 h2 = __floats2bfloat162_rn((x[e + 2 * k] - mean) * inv * sc[2 * k],
                                                          (x[e + 2 * k + 1] - mean) * inv * sc[2 * k + 1]);
          pw[k] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        *reinterpret_cast<uint4*>(op + e) = pk;
      }
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) op[e] = __float2bfloat16((x[e] - mean) * inv * a.ln_scale[lane * E + e]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const uint32_t j = lane + 32 * e;
      if (j < d) a.out[(size_t)row * d + j] = __float2bfloat16((x[e] - mean) * inv * a.ln_scale[j]);
    }
  }
}

// Row-block form (the common shapes: d % 32 == 0, H in {1, 2, 4, 8}, D % 4 == 0):
// one CTA per 32 query rows of one request's query tile. Warp w owns the d/8
// columns [w d/8, (w+1) d/8) (one head), lane = row, so every partial-slot
// read is one 4-column chunk of 32 consecutive rows = 512 contiguous bytes
// (the chunked slot layout, part_index); the gate operand u is staged through
// shared memory with row-contiguous loads, the row statistics are reduced
// across the 8 warps in shared memory, and the normalised rows leave through
// shared memory as row-contiguous 16-B stores. The request / segment / slot
// metadata is loaded once per block instead of once per row.
constexpr int GB_WARPS = 8;
bool gate_block_supported(uint32_t H, uint32_t D) {
  const uint32_t d = H * D;
  return d % 32 == 0 && d <= 512 && D % 4 == 0 && (H == 1 || H == 2 || H == 4 || H == 8);
}

template <int CPW>  // 4-column chunks per warp (d / 32)
__global__ void __launch_bounds__(GB_WARPS * 32, 4) gate_block_kernel(GateArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int NC = CPW * 4;                      // columns per warp
  constexpr int d = NC * GB_WARPS;
  constexpr int UP = d + 8;                        // padded bf16 row stride in shared memory
  __shared__ __align__(16) __nv_bfloat16 s_u[kGateBlockRows * UP];  // u rows, later the output rows
  __shared__ float s_red[GB_WARPS][kGateBlockRows];
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t req = a.blocks[2 * blockIdx.x], i0 = a.blocks[2 * blockIdx.x + 1];
  const ReqDev R = a.reqs[req];
  const uint32_t nrows = min(kGateBlockRows, R.n_q - i0);
  const size_t row0 = size_t(R.q_row0) + i0;       // global row of block row 0
  // stage u (row-contiguous 16-B loads)
  constexpr int V16 = d / 8;                       // 16-B vectors per row
  for (uint32_t v = threadIdx.x; v < kGateBlockRows * V16; v += GB_WARPS * 32) {
    const uint32_t rr = v / V16, cv = v % V16;
    uint4 x = make_uint4(0, 0, 0, 0);
    if (rr < nrows) x = *reinterpret_cast<const uint4*>(a.u + (row0 + rr) * d + cv * 8);
    *reinterpret_cast<uint4*>(s_u + rr * UP + cv * 8) = x;
  }
  // merge this warp's head's partial slots for row `lane`
  const uint32_t c0 = warp * NC, h = c0 / a.D, cd = c0 % a.D;   // first column, head, column within the head
  const uint32_t qt = i0 / a.bm, ri = i0 % a.bm + lane;
  const AttnSeg sg = a.segs[R.seg0 + h * R.qtiles + qt];
  const bool valid = lane < nrows;
  // the slots' log-sum-exps (up to 4 held in registers: one batch of independent
  // loads; longer segments reload them), then every slot's chunks issued
  // without a dependence on the previous slot's
  float lk[4];
  float mx = -INFINITY;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    lk[k] = k < int(sg.n_parts) ? a.part_lse[size_t(sg.part_base + k) * a.bm + ri] : -INFINITY;
    mx = fmaxf(mx, lk[k]);
  }
  for (uint32_t k = 4; k < sg.n_parts; ++k) mx = fmaxf(mx, a.part_lse[size_t(sg.part_base + k) * a.bm + ri]);
  float acc[NC];
#pragma unroll
  for (int e = 0; e < NC; ++e) acc[e] = 0.f;
  float den = 0.f;
  for (uint32_t k = 0; k < sg.n_parts; ++k) {
    const float l = k < 4 ? lk[k & 3] : a.part_lse[size_t(sg.part_base + k) * a.bm + ri];
    const float w = (valid && l != -INFINITY) ? exp2f(l - mx) : 0.f;  // an empty slot row weighs 0
    den += w;
    const float* src = a.part_o + part_index(sg.part_base + k, a.bm, ri, cd, a.D);
    float4 v[CPW];
#pragma unroll
    for (int c = 0; c < CPW; ++c)
      v[c] = w != 0.f ? *reinterpret_cast<const float4*>(src + size_t(c) * a.bm * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      acc[4 * c] += w * v[c].x; acc[4 * c + 1] += w * v[c].y; acc[4 * c + 2] += w * v[c].z; acc[4 * c + 3] += w * v[c].w;
    }
  }
  __syncthreads();  // u staged
  const float inv_den = den > 0.f ? 1.f / den : 0.f;
  float sum = 0.f;
#pragma unroll
  for (int e = 0; e < NC; e += 2) {
    const float2 u2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(s_u + lane * UP + c0 + e));
    acc[e] = silu_f(acc[e] * inv_den) * u2.x;
    acc[e + 1] = silu_f(acc[e + 1] * inv_den) * u2.y;
    sum += acc[e] + acc[e + 1];
  }
  s_red[warp][lane] = sum;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < GB_WARPS; ++w) tot += s_red[w][lane];
  const float mean = tot / float(d);
  float var = 0.f;
#pragma unroll
  for (int e = 0; e < NC; ++e) { const float c = acc[e] - mean; var += c * c; }
  __syncthreads();  // everyone read the sums
  s_red[warp][lane] = var;
  __syncthreads();
  float vt = 0.f;
#pragma unroll
  for (int w = 0; w < GB_WARPS; ++w) vt += s_red[w][lane];
  const float rstd = 1.0f / sqrtf(vt / float(d) + 1e-6f);
  // normalised row -> shared memory (over u, which every thread has read), then out
#pragma unroll
  for (int e = 0; e < NC; e += 2) {
    const float2 sc = *reinterpret_cast<const float2*>(a.ln_scale + c0 + e);
    *reinterpret_cast<__nv_bfloat162*>(s_u + lane * UP + c0 + e) =
        __floats2bfloat162_rn((acc[e] - mean) * rstd * sc.x, (acc[e + 1] - mean) * rstd * sc.y);
  }
  __syncthreads();
  for (uint32_t v = threadIdx.x; v < kGateBlockRows * V16; v += GB_WARPS * 32) {
    const uint32_t rr = v / V16, cv = v % V16;
    if (rr < nrows) *reinterpret_cast<uint4*>(a.out + (row0 + rr) * d + cv * 8) = *reinterpret_cast<const uint4*>(s_u + rr * UP + cv * 8);
  }
}

void launch_gate_norm(const GateArgs& a, cudaStream_t s) {
  if (a.rows == 0) return;
  const uint32_t d = a.H * a.D, E = d % 32 == 0 ? d / 32 : 0;
  static const bool rows_only = [] {  // MTKV_GATE=row: the row-per-warp kernel everywhere (A/B switch)
    const char* e = std::getenv("MTKV_GATE");
    return e && e[0] == 'r';
  }();
  // row blocks pay off once there are several per SM (prefill-shaped batches:
  // 75.6 vs 105.6 us per launch); small decode batches keep one warp per row
  // (10.7 vs 12.5 us) — ncu launch lists of the configs[1] bench, both policies
  if (!rows_only && a.blocks && a.n_blocks >= 4 * uint32_t(num_sms()) && gate_block_supported(a.H, a.D)) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.n_blocks);
    cfg.blockDim = dim3(GB_WARPS * 32);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    switch (d / 32) {
      case 1: cudaLaunchKernelEx(&cfg, gate_block_kernel<1>, a); return;
      case 2: cudaLaunchKernelEx(&cfg, gate_block_kernel<2>, a); return;
      case 4: cudaLaunchKernelEx(&cfg, gate_block_kernel<4>, a); return;
      case 8: cudaLaunchKernelEx(&cfg, gate_block_kernel<8>, a); return;
      case 16: cudaLaunchKernelEx(&cfg, gate_block_kernel<16>, a); return;
      default: break;  // other widths: the row-per-warp kernel below
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.rows + GATE_WARPS - 1) / GATE_WARPS);
  cfg.blockDim = dim3(GATE_WARPS * 32);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (E && a.D % E == 0) {
    switch (E) {
      case 1: cudaLaunchKernelEx(&cfg, gate_norm_kernel<1>, a); return;
      case 2: cudaLaunchKernelEx(&cfg, gate_norm_kernel<2>, a); return;
      case 4: cudaLaunchKernelEx(&cfg, gate_norm_kernel<4>, a); return;
      case 8: cudaLaunchKernelEx(&cfg, gate_norm_kernel<8>, a); return;
      case 16: cudaLaunchKernelEx(&cfg, gate_norm_kernel<16>, a); return;
      default: break;
    }
  }
  cudaLaunchKernelEx(&cfg, gate_norm_kernel<0>, a);
}

// -------------------------------------------------------- scatter/gather ---
// One CTA per (chunk, layer, K|V, page of the chunk): a contiguous
// page_size*d segment; 128-bit loads/stores when aligned.
template <bool TO_POOL>
__global__ void chunk_copy_kernel(__nv_bfloat16* pool, __nv_bfloat16* staging, const ChunkWork* work,
                                  const uint32_t* pages, PoolGeom g) {
  const uint32_t ppc = g.chunk / g.S;
  uint32_t b = blockIdx.x;
  const uint32_t p = b % ppc; b /= ppc;
  const uint32_t kv = b % 2; b /= 2;
  const uint32_t l = b % g.L; b /= g.L;
  const ChunkWork w = work[b];
  const uint32_t page = pages[w.pages_off + p];
  const size_t seg = (size_t)g.S * g.d;
  __nv_bfloat16* pp = pool + g.off(l, page, kv, 0);
  __nv_bfloat16* sp = staging + ((((size_t)w.slot * g.L + l) * 2 + kv) * g.chunk + (size_t)p * g.S) * g.d;
  if ((seg % 8) == 0) {
    // all loads of a thread in flight before its stores (8 x 16 B per thread)
    constexpr int U = 8;
    uint4* dst = reinterpret_cast<uint4*>(TO_POOL ? pp : sp);
    const uint4* src = reinterpret_cast<const uint4*>(TO_POOL ? sp : pp);
    const size_t n = seg / 8;
    for (size_t base = threadIdx.x; base < n; base += (size_t)blockDim.x * U) {
      uint4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t idx = base + (size_t)u * blockDim.x;
        if (idx < n) r[u] = __ldcs(src + idx);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t idx = base + (size_t)u * blockDim.x;
        if (idx < n) dst[idx] = r[u];
      }
    }
  } else {
    __nv_bfloat16* dst = TO_POOL ? pp : sp;
    const __nv_bfloat16* src = TO_POOL ? sp : pp;
    for (size_t i = threadIdx.x; i < seg; i += blockDim.x) dst[i] = src[i];
  }
}

void launch_scatter_chunks(__nv_bfloat16* pool, const __nv_bfloat16* staging, const ChunkWork* work,
                           const uint32_t* pages, uint32_t n_chunks, const PoolGeom& g, cudaStream_t s) {
  if (!n_chunks) return;
  const uint32_t blocks = n_chunks * g.L * 2 * (g.chunk / g.S);
  chunk_copy_kernel<true><<<blocks, 128, 0, s>>>(pool, const_cast<__nv_bfloat16*>(staging), work, pages, g);
}

void launch_gather_chunks(__nv_bfloat16* staging, const __nv_bfloat16* pool, const ChunkWork* work,
                          const uint32_t* pages, uint32_t n_chunks, const PoolGeom& g, cudaStream_t s) {
  if (!n_chunks) return;
  const uint32_t blocks = n_chunks * g.L * 2 * (g.chunk / g.S);
  chunk_copy_kernel<false><<<blocks, 128, 0, s>>>(const_cast<__nv_bfloat16*>(pool), staging, work, pages, g);
}

// -------------------------------------------------------------- tag mode ---
__global__ void tag_append_kernel(__nv_bfloat16* pool, const ReqDev* reqs, const uint32_t* pages, PoolGeom g) {
  const ReqDev R = reqs[blockIdx.y];
  for (uint32_t i = blockIdx.x; i < R.n_hist; i += gridDim.x) {
    const uint64_t pos = R.start + i;
    const uint32_t page = pages[R.pages_off + (uint32_t)(pos / g.S)], slot = (uint32_t)(pos % g.S);
    for (uint32_t l = 0; l < g.L; ++l)
      for (uint32_t kv = 0; kv < 2; ++kv) {
        uint16_t* dst = reinterpret_cast<uint16_t*>(pool + g.off(l, page, kv, slot));
        for (uint32_t j = threadIdx.x; j < g.d; j += blockDim.x) dst[j] = tag_word(R.user, pos, l, kv, j);
      }
  }
}

void launch_tag_append(__nv_bfloat16* pool, const ReqDev* reqs, const uint32_t* pages, uint32_t n_reqs,
                       uint32_t max_hist, const PoolGeom& g, cudaStream_t s) {
  if (!n_reqs || !max_hist) return;
  dim3 grid(max_hist < 256 ? max_hist : 256, n_reqs);
  tag_append_kernel<<<grid, 64, 0, s>>>(pool, reqs, pages, g);
}

}  // namespace mtkv_b200
