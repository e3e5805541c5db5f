// MUFU.EX2 vs FMA-pipe exp2 throughput on one SM (diagnostic microbenchmark).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_rate mufu_rate.cu && ./mufu_rate
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float ex2p(float x) {
  const float xc = fmaxf(x, -126.f);
  const float t = xc + 12582912.f;
  const int j = __float_as_int(t) - 0x4B400000;
  const float f = xc - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.0551716566f, f, 0.2426111399f), f, 0.6932609894f), f, 0.9999280726f);
  return __int_as_float(__float_as_int(p) + (j << 23));
}
template <int POLY>
__global__ void k(float* out, long long* cyc, int iters) {
  float v[64];
  for (int i = 0; i < 64; ++i) v[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = (POLY && i % POLY == POLY - 1) ? ex2p(v[i] - 1.f) : ex2(v[i] - 1.f);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 64; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int POLY> void run(int warps) {
  float* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 1024);
  const int iters = 200;
  k<POLY><<<1, warps * 32>>>(o, c, iters);
  k<POLY><<<1, warps * 32>>>(o, c, iters);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double exps = double(iters) * 64 * warps * 32;
  printf("poly=%d warps=%2d: %.2f exps/clk/SM (%.1f cycles per 64-exp row-block per warp-pair-per-SMSP)\n", POLY, warps,
         exps / h, double(h) / iters);
}
int main() {
  for (int w : {4, 8, 16}) { run<0>(w); run<8>(w); run<4>(w); run<3>(w); run<2>(w); }
  return 0;
}
