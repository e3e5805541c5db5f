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

// out[i][h*D + c] = log-sum-exp merge (base 2) of segment (h, i / bm)'s partial slots
__global__ void merge_segs_kernel(float* out, const float* part, const float* lse, const AttnSeg* segs, uint32_t n_q,
                                  uint32_t H, uint32_t D, uint32_t bm, uint32_t qtiles) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x, d = H * D;
  if (idx >= n_q * d) return;
  const uint32_t i = idx / d, j = idx % d, h = j / D, c = j % D, ri = i % bm;
  const AttnSeg sg = segs[h * qtiles + i / bm];
  float m = -INFINITY;
  for (uint32_t k = 0; k < sg.n_parts; ++k) m = fmaxf(m, lse[size_t(sg.part_base + k) * bm + ri]);
  float num = 0.f, den = 0.f;
  for (uint32_t k = 0; k < sg.n_parts; ++k) {
    const size_t prow = size_t(sg.part_base + k) * bm + ri;
    if (lse[prow] == -INFINITY) continue;
    const float w = exp2f(lse[prow] - m);
    num += w * part[prow * D + c];
    den += w;
  }
  out[idx] = den > 0.f ? num / den : 0.f;
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
  const char* force = std::getenv("MTKV_ATTN");
  const bool tc = attn_tc_supported(g) && !(force && std::string(force) == "mma");
  AttnPlan plan;
  plan_attention(&r, 1, g, tc, tc ? uint32_t(num_sms()) : 0, plan);
  const uint32_t n_items = tc ? plan.n_ctas() : uint32_t(plan.items.size());
  // one device allocation: request | segments | items or pieces + CTA offsets | lse | partials
  size_t off = 0;
  auto carve = [&](size_t bytes) { const size_t o = off; off = (off + bytes + 255) & ~size_t(255); return o; };
  const size_t o_req = carve(sizeof(ReqDev));
  const size_t o_seg = carve(plan.segs.size() * sizeof(AttnSeg));
  const size_t o_items = carve(plan.items.size() * sizeof(AttnItem));
  const size_t o_pieces = carve(plan.pieces.size() * sizeof(AttnPiece));
  const size_t o_cta = carve(plan.cta_off.size() * sizeof(uint32_t));
  const size_t o_lse = carve(size_t(plan.n_slots) * plan.bm * sizeof(float));
  const size_t o_part = carve(size_t(plan.n_slots) * plan.bm * g.D * sizeof(float));
  char* buf = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&buf, off, s);
  if (e != cudaSuccess) return finish(e);
  auto up = [&](size_t o, const void* src, size_t bytes) {
    if (e == cudaSuccess && bytes) e = cudaMemcpyAsync(buf + o, src, bytes, cudaMemcpyHostToDevice, s);
  };
  up(o_req, &r, sizeof(r));
  up(o_seg, plan.segs.data(), plan.segs.size() * sizeof(AttnSeg));
  up(o_items, plan.items.data(), plan.items.size() * sizeof(AttnItem));
  up(o_pieces, plan.pieces.data(), plan.pieces.size() * sizeof(AttnPiece));
  up(o_cta, plan.cta_off.data(), plan.cta_off.size() * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // host plan vectors die with this scope
  AttnArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.pool = static_cast<const __nv_bfloat16*>(pool);
  a.pages = d_pages;
  a.reqs = reinterpret_cast<const ReqDev*>(buf + o_req);
  a.segs = reinterpret_cast<const AttnSeg*>(buf + o_seg);
  a.items = reinterpret_cast<const AttnItem*>(buf + o_items);
  a.pieces = reinterpret_cast<const AttnPiece*>(buf + o_pieces);
  a.cta_off = reinterpret_cast<const uint32_t*>(buf + o_cta);
  a.n_items = n_items;
  a.part_o = reinterpret_cast<float*>(buf + o_part);
  a.part_lse = reinterpret_cast<float*>(buf + o_lse);
  a.g = g;
  a.layer = layer;
  a.bq = plan.bm;
  a.scale_log2 = float(1.4426950408889634 / sqrt(double(g.D)));
  if (e == cudaSuccess) {
    if (tc) {
      alignas(64) CUtensorMap pmap, qmap;
      if (make_pool_map(&pmap, pool, g) || make_q_map(&qmap, q, n_q, g)) {
        cudaFreeAsync(buf, s);
        set_last_error("paged_attention: cuTensorMapEncodeTiled failed");
        return MTKV_ERROR;
      }
      launch_attention_tc(pmap, qmap, a, s);
    } else {
      launch_attention(a, s);
    }
    merge_segs_kernel<<<(n_q * g.d + 255) / 256, 256, 0, s>>>(out, a.part_o, a.part_lse, a.segs, n_q, g.H, g.D,
                                                               plan.bm, r.qtiles);
  }
  cudaFreeAsync(buf, s);
  return finish(e);
}

}  // extern "C"
