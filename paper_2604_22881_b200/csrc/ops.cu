// Raw device ops of the C-ABI (kernel-level parity tests and integrations that
// own their buffers): chunk scatter/gather and single-request paged attention.
#include <cmath>
#include <cstdlib>
#include <string>

#include "kernels.cuh"
#include "../../include/mtkv_b200.h"

namespace mtkv_b200 {
void set_last_error(const std::string& m);
}

using namespace mtkv_b200;

static PoolGeom geom(const mtkv_kv_config* kv, uint32_t num_pages) {
  PoolGeom g{};
  g.L = kv->num_layers;
  g.H = kv->num_heads;
  g.D = kv->head_dim;
  g.d = kv->num_heads * kv->head_dim;
  g.S = kv->page_size;
  g.chunk = kv->chunk_size;
  g.num_pages = num_pages;
  return g;
}

static int finish(cudaError_t e) {
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_error(std::string("device op: ") + cudaGetErrorString(e));
    return MTKV_ERROR;
  }
  return MTKV_OK;
}

static int chunk_op(bool to_pool, void* pool, void* staging, const uint32_t* d_page_ids, uint32_t n_chunks,
                    const mtkv_kv_config* kv, uint32_t num_pages, void* stream) {
  if (!n_chunks) return MTKV_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const PoolGeom g = geom(kv, num_pages);
  const uint32_t ppc = g.chunk / g.S;
  ChunkWork* work = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&work, n_chunks * sizeof(ChunkWork), s);
  if (e != cudaSuccess) return finish(e);
  ChunkWork* h = new ChunkWork[n_chunks];
  for (uint32_t c = 0; c < n_chunks; ++c) h[c] = ChunkWork{c, c * ppc};
  e = cudaMemcpyAsync(work, h, n_chunks * sizeof(ChunkWork), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  delete[] h;
  if (to_pool)
    launch_scatter_chunks(static_cast<__nv_bfloat16*>(pool), static_cast<const __nv_bfloat16*>(staging), work,
                          d_page_ids, n_chunks, g, s);
  else
    launch_gather_chunks(static_cast<__nv_bfloat16*>(staging), static_cast<const __nv_bfloat16*>(pool), work,
                         d_page_ids, n_chunks, g, s);
  cudaFreeAsync(work, s);
  return finish(e);
}

// out = merge of the two pipeline partials (log-sum-exp weights, base 2)
__global__ void merge2_kernel(float* out, const float* part, const float* lse, uint32_t n_q, uint32_t H,
                              uint32_t D) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x, d = H * D;
  if (idx >= n_q * d) return;
  const uint32_t i = idx / d, j = idx % d, h = j / D;
  const float l0 = lse[size_t(i) * H + h], l1 = lse[(size_t(n_q) + i) * H + h];
  const float m = fmaxf(l0, l1);
  const float w0 = l0 == -INFINITY ? 0.f : exp2f(l0 - m), w1 = l1 == -INFINITY ? 0.f : exp2f(l1 - m);
  const float den = w0 + w1;
  out[idx] = den > 0.f ? (w0 * part[idx] + w1 * part[size_t(n_q) * d + idx]) / den : 0.f;
}

extern "C" {

int mtkv_op_scatter_chunks(void* pool, const void* staging, const uint32_t* d_page_ids, uint32_t n_chunks,
                           const mtkv_kv_config* kv, uint32_t num_pages, void* stream) {
  return chunk_op(true, pool, const_cast<void*>(staging), d_page_ids, n_chunks, kv, num_pages, stream);
}

int mtkv_op_gather_chunks(void* staging, const void* pool, const uint32_t* d_page_ids, uint32_t n_chunks,
                          const mtkv_kv_config* kv, uint32_t num_pages, void* stream) {
  return chunk_op(false, const_cast<void*>(pool), staging, d_page_ids, n_chunks, kv, num_pages, stream);
}

int mtkv_op_paged_attention(float* out, const void* q, const void* pool, const uint32_t* d_pages, uint32_t n_q,
                            uint64_t p_pre, uint64_t n_keys, uint32_t layer, const mtkv_kv_config* kv,
                            uint32_t num_pages, void* stream) {
  if (n_keys != p_pre + n_q) {
    set_last_error("paged_attention: n_keys must equal p_pre + n_q");
    return MTKV_ERROR;
  }
  if (!n_q) return MTKV_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const PoolGeom g = geom(kv, num_pages);
  ReqDev r{};
  r.q_row0 = 0;
  r.n_q = n_q;
  r.n_hist = n_q;
  r.n_cand = 0;
  r.start = p_pre;
  r.pages_off = 0;
  r.n_pages = uint32_t((n_keys + g.S - 1) / g.S);
  r.part_base = 0;
  r.split_keys = 0xFFFFFF00u;
  const char* force = std::getenv("MTKV_ATTN");
  const bool tc = attn_tc_supported(g) && !(force && std::string(force) == "mma");
  r.n_splits = tc ? 2 : 1;  // the tcgen05 kernel emits one partial per softmax pipeline
  const uint32_t bq = (tc || n_q > 64) ? 128 : 64;
  const uint32_t qtiles = (n_q + bq - 1) / bq, n_items = g.H * qtiles;
  AttnItem* hi = new AttnItem[n_items];
  uint32_t k = 0;
  for (uint32_t h = 0; h < g.H; ++h)
    for (uint32_t t = 0; t < qtiles; ++t) hi[k++] = AttnItem{0, h, t, 0};
  char* buf = nullptr;
  const size_t part_bytes = tc ? size_t(2) * n_q * g.d * sizeof(float) : 0;
  const size_t bytes = 256 + n_items * sizeof(AttnItem) + size_t(2) * n_q * g.H * sizeof(float) + part_bytes;
  cudaError_t e = cudaMallocAsync((void**)&buf, bytes, s);
  if (e != cudaSuccess) { delete[] hi; return finish(e); }
  ReqDev* dr = reinterpret_cast<ReqDev*>(buf);
  AttnItem* di = reinterpret_cast<AttnItem*>(buf + 256);
  float* lse = reinterpret_cast<float*>(buf + 256 + n_items * sizeof(AttnItem));
  float* part = tc ? lse + size_t(2) * n_q * g.H : nullptr;
  e = cudaMemcpyAsync(dr, &r, sizeof(r), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(di, hi, n_items * sizeof(AttnItem), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  delete[] hi;
  AttnArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.pool = static_cast<const __nv_bfloat16*>(pool);
  a.pages = d_pages;
  a.reqs = dr;
  a.items = di;
  a.n_items = n_items;
  a.part_o = tc ? part : out;
  a.part_lse = lse;
  a.g = g;
  a.layer = layer;
  a.bq = bq;
  a.scale_log2 = float(1.4426950408889634 / sqrt(double(g.D)));
  if (e == cudaSuccess) {
    if (tc) {
      alignas(64) CUtensorMap map;
      if (make_pool_map(&map, pool, g)) {
        cudaFreeAsync(buf, s);
        set_last_error("paged_attention: cuTensorMapEncodeTiled failed");
        return MTKV_ERROR;
      }
      launch_attention_tc(map, a, s);
      merge2_kernel<<<(n_q * g.d + 255) / 256, 256, 0, s>>>(out, part, lse, n_q, g.H, g.D);
    } else {
      launch_attention(a, s);
    }
  }
  cudaFreeAsync(buf, s);
  return finish(e);
}

}  // extern "C"
