// Raw device ops of the C-ABI (kernel-level parity tests and integrations that
// own their buffers): chunk scatter/gather and single-request paged attention.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

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

// out[row][h*D + c] = log-sum-exp merge (base 2) of the partial slots of the
// row's segment (request, head, query tile)
__global__ void merge_segs_kernel(float* out, const float* part, const float* lse, const AttnSeg* segs,
                                  const ReqDev* reqs, const uint32_t* row_req, uint32_t rows, uint32_t H, uint32_t D,
                                  uint32_t bm) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x, d = H * D;
  if (idx >= rows * d) return;
  const uint32_t row = idx / d, j = idx % d, h = j / D, c = j % D;
  const ReqDev R = reqs[row_req[row]];
  const uint32_t i = row - R.q_row0, ri = i % bm;
  const AttnSeg sg = segs[R.seg0 + h * R.qtiles + i / bm];
  float m = -INFINITY;
  for (uint32_t k = 0; k < sg.n_parts; ++k) m = fmaxf(m, lse[size_t(sg.part_base + k) * bm + ri]);
  float num = 0.f, den = 0.f;
  for (uint32_t k = 0; k < sg.n_parts; ++k) {
    const size_t prow = size_t(sg.part_base + k) * bm + ri;
    if (lse[prow] == -INFINITY) continue;
    const float w = exp2f(lse[prow] - m);
    num += w * part[part_index(sg.part_base + k, bm, ri, c, D)];
    den += w;
  }
  out[idx] = den > 0.f ? num / den : 0.f;
}

// Batched paged attention: request r's fresh rows [q_row0, q_row0 + n_q[r]) of q
// attend over its p_pre[r] cached keys + themselves (causal); its page list
// starts at d_pages[page_off[r]].
static int attention_batch(float* out, const void* q, const void* pool, const uint32_t* d_pages,
                           const uint32_t* page_off, const uint32_t* n_q, const uint64_t* p_pre, uint32_t n_req,
                           uint32_t layer, const mtkv_kv_config* kv, uint32_t num_pages, uint32_t repeat,
                           float* ms_per_launch, cudaStream_t s) {
  const PoolGeom g = geom(kv, num_pages);
  std::vector<ReqDev> rq(n_req);
  uint32_t rows = 0;
  for (uint32_t r = 0; r < n_req; ++r) {
    ReqDev& x = rq[r];
    x = ReqDev{};
    x.q_row0 = rows;
    x.n_q = x.n_hist = n_q[r];
    x.start = p_pre[r];
    x.dep_start = p_pre[r];
    x.pages_off = page_off[r];
    x.n_pages = uint32_t((p_pre[r] + n_q[r] + g.S - 1) / g.S);
    rows += n_q[r];
  }
  if (!rows) return MTKV_OK;
  std::vector<uint32_t> row_req(rows);
  for (uint32_t r = 0; r < n_req; ++r)
    for (uint32_t i = 0; i < n_q[r]; ++i) row_req[rq[r].q_row0 + i] = r;
  const AttnKind kind = attn_kind(g);
  const bool tc = kind != AttnKind::Mma;
  AttnPlan plan;
  plan_attention(rq.data(), n_req, g, tc, attn_plan_ctas(kind, num_sms()), plan,
                 kind == AttnKind::Tc && attn_pair_wanted(g, rq.data(), n_req));
  if (kind == AttnKind::Pp && plan.n_ctas() % 2) plan.cta_off.push_back(plan.cta_off.back());
  const uint32_t n_items = tc ? plan.n_ctas() : uint32_t(plan.items.size());
  // one device allocation: requests | rows | segments | items or pieces + CTA offsets | lse | partials
  size_t off = 0;
  auto carve = [&](size_t bytes) { const size_t o = off; off = (off + bytes + 255) & ~size_t(255); return o; };
  const size_t o_req = carve(rq.size() * sizeof(ReqDev));
  const size_t o_rr = carve(row_req.size() * sizeof(uint32_t));
  const size_t o_seg = carve(plan.segs.size() * sizeof(AttnSeg));
  const size_t o_items = carve(plan.items.size() * sizeof(AttnItem));
  const size_t o_pieces = carve(plan.pieces.size() * sizeof(AttnPiece));
  const size_t o_cta = carve(plan.cta_off.size() * sizeof(uint32_t));
  const size_t o_lse = carve(size_t(plan.n_slots) * plan.bm * sizeof(float));
  const size_t o_part = carve(size_t(plan.n_slots) * part_slot_floats(plan.bm, g.D) * sizeof(float));
  char* buf = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&buf, off, s);
  if (e != cudaSuccess) return finish(e);
  auto up = [&](size_t o, const void* src, size_t bytes) {
    if (e == cudaSuccess && bytes) e = cudaMemcpyAsync(buf + o, src, bytes, cudaMemcpyHostToDevice, s);
  };
  up(o_req, rq.data(), rq.size() * sizeof(ReqDev));
  up(o_rr, row_req.data(), row_req.size() * sizeof(uint32_t));
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
  a.pair = plan.pair;
  a.scale_log2 = float(1.4426950408889634 / sqrt(double(g.D)));
  if (e == cudaSuccess) {
    alignas(64) CUtensorMap pmap, qmap;
    if (tc && (make_pool_map(&pmap, pool, g) || make_q_map(&qmap, q, rows, g))) {
      cudaFreeAsync(buf, s);
      set_last_error("paged_attention: cuTensorMapEncodeTiled failed");
      return MTKV_ERROR;
    }
    // MTKV_ATTN_TRACE=<file>: per-CTA event timelines of the last launch (tools/attn_trace.py)
    const char* trace_path = tc ? std::getenv("MTKV_ATTN_TRACE") : nullptr;
    unsigned long long* trace = nullptr;
    const size_t trace_bytes = size_t(kTraceCtas) * kTraceKinds * kTraceTiles * 8;
    if (trace_path && cudaMallocAsync((void**)&trace, trace_bytes, s) == cudaSuccess) {
      cudaMemsetAsync(trace, 0, trace_bytes, s);
      a.trace = trace;
    }
    // repeat > 1: launch 0 is the warm-up; launches 1..repeat-1 are timed one by
    // one with CUDA events, each after a 256 MB memset that evicts L2 (so a
    // launch never reuses K/V the previous launch left in the 126 MB L2)
    std::vector<cudaEvent_t> ev;
    void* flush = nullptr;
    if (repeat > 1 && ms_per_launch) {
      ev.resize(2 * (repeat - 1));
      for (auto& x : ev) cudaEventCreate(&x);
      cudaMallocAsync(&flush, size_t(256) << 20, s);
    }
    for (uint32_t it = 0; it < std::max<uint32_t>(repeat, 1); ++it) {
      if (it >= 1 && !ev.empty()) {
        cudaMemsetAsync(flush, int(it & 0xFF), size_t(256) << 20, s);
        cudaEventRecord(ev[2 * (it - 1)], s);
      }
      launch_attention_any(kind, pmap, qmap, a, s);
      if (it >= 1 && !ev.empty()) cudaEventRecord(ev[2 * (it - 1) + 1], s);
    }
    if (!ev.empty()) {
      cudaStreamSynchronize(s);
      double tot = 0;
      for (uint32_t it = 1; it < repeat; ++it) {
        float ms = 0;
        cudaEventElapsedTime(&ms, ev[2 * (it - 1)], ev[2 * (it - 1) + 1]);
        tot += ms;
      }
      *ms_per_launch = float(tot / double(repeat - 1));
      for (auto& x : ev) cudaEventDestroy(x);
      cudaFreeAsync(flush, s);
    }
    if (trace) {
      std::vector<unsigned long long> h(trace_bytes / 8);
      cudaMemcpyAsync(h.data(), trace, trace_bytes, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      if (FILE* f = std::fopen(trace_path, "wb")) {
        std::fwrite(h.data(), 8, h.size(), f);
        std::fclose(f);
      }
      cudaFreeAsync(trace, s);
    }
    merge_segs_kernel<<<(rows * g.d + 255) / 256, 256, 0, s>>>(out, a.part_o, a.part_lse, a.segs, a.reqs,
                                                                reinterpret_cast<const uint32_t*>(buf + o_rr), rows,
                                                                g.H, g.D, plan.bm);
  }
  cudaFreeAsync(buf, s);
  return finish(e);
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
  const uint32_t zero = 0;
  return attention_batch(out, q, pool, d_pages, &zero, &n_q, &p_pre, 1, layer, kv, num_pages, 1, nullptr,
                         static_cast<cudaStream_t>(stream));
}

int mtkv_op_paged_attention_batch(float* out, const void* q, const void* pool, const uint32_t* d_pages,
                                  const uint32_t* page_off, const uint32_t* n_q, const uint64_t* p_pre, uint32_t n_req,
                                  uint32_t layer, const mtkv_kv_config* kv, uint32_t num_pages, uint32_t repeat,
                                  float* ms_per_launch, void* stream) {
  return attention_batch(out, q, pool, d_pages, page_off, n_q, p_pre, n_req, layer, kv, num_pages, repeat,
                         ms_per_launch, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

// Dense layer of the GR block (model.cpp:71 matmul, with the silu of :174/:191
// when act = 1): out[M x N] bf16 = act(a[M x K] . w[K x N]), fp32 accumulation.
// The tcgen05 kernel runs whenever it covers the shape (K, N multiples of 64),
// the mma.sync kernel otherwise; tc = 1 refuses shapes the tcgen05 kernel does
// not cover instead of falling back. a_rows_alloc: rows allocated behind `a`.
extern "C" int mtkv_op_dense(void* out, const void* a, const void* w, uint32_t M, uint32_t N, uint32_t K,
                             uint64_t a_rows_alloc, int act, int tc, void* stream) {
  GemmArgs g{};
  g.A = static_cast<const __nv_bfloat16*>(a);
  g.B = static_cast<const __nv_bfloat16*>(w);
  g.M = int(M);
  g.N = int(N);
  g.K = int(K);
  g.epi = act ? Epi::SiluBf16 : Epi::Bf16;
  g.out = out;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (gemm_tc_supported(g)) {
    if (launch_gemm_tc(g, a_rows_alloc < M ? M : a_rows_alloc, s)) {
      set_last_error("dense: cuTensorMapEncodeTiled failed");
      return MTKV_ERROR;
    }
  } else if (tc) {
    set_last_error("dense: shape not covered by the tcgen05 kernel (K and N must be multiples of 64)");
    return MTKV_ERROR;
  } else {
    launch_gemm(g, s);
  }
  return finish(cudaSuccess);
}
