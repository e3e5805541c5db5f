// Device-side data structures shared by the executor and the kernels.
//
// HBM layout of the paged store (paper §4.1, reference store.hpp:54):
//   pool[L][num_pages][2 (K,V)][page_size][H*D] bf16
// A page id addresses the same slot in every layer plane. Host chunks and the
// onload staging slots use [L][2][chunk_size][H*D] bf16, so one chunk is one
// contiguous copy-engine transfer.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace mtkv_b200 {

struct PoolGeom {
  uint32_t L, H, D, d, S;  // layers, heads, head dim, hidden, page size
  uint32_t num_pages;      // device pages + transient (recompute) pages
  uint32_t chunk;          // chunk size (tokens)
  // element offset of (layer, page, kv, slot)
  __host__ __device__ inline uint64_t off(uint32_t l, uint32_t page, uint32_t kv, uint32_t slot) const {
    return ((((uint64_t)l * num_pages + page) * 2 + kv) * S + slot) * d;
  }
};

// Per-request record uploaded with each batch.
struct ReqDev {
  uint32_t q_row0;      // first fresh row of this request in the batch
  uint32_t n_q;         // fresh rows: n_hist history rows then n_cand candidate rows
  uint32_t n_hist;
  uint32_t n_cand;
  uint64_t start;       // position of the first fresh row (= cached prefix length)
  uint32_t pages_off, n_pages;      // user pages (positions 0 .. start+n_hist-1)
  uint32_t scratch_off, n_scratch;  // candidate pages
  uint32_t part_base;   // first partial row of this request (split-K attention)
  uint32_t n_splits;
  uint32_t split_keys;
  uint32_t user;
};

struct AttnItem {  // one CTA of the attention kernel
  uint32_t req, head, qtile, split;
};

struct ChunkWork {  // one staged/offloaded chunk
  uint32_t slot;       // staging / offload slot
  uint32_t pages_off;  // pages_per_chunk page ids in the batch page array
};

// Launchers (kernels.cu). All take the stream to enqueue on.
enum class Epi { Proj = 0, SiluBf16 = 1, Bf16 = 2, F32 = 3 };

struct GemmArgs {
  const __nv_bfloat16* A;   // [M x K] (row r read from row_idx[r] if row_idx)
  const uint32_t* row_idx;  // optional A-row gather
  const __nv_bfloat16* B;   // [K x N] row-major (reference weight layout)
  int M, N, K;
  Epi epi;
  void* out;                // Bf16/SiluBf16: bf16 [M x N]; F32: float [M x N]
  // Proj epilogue: silu, then u -> out_u, q -> out_q, k/v -> pool at kv_off[r]
  __nv_bfloat16* out_u;
  __nv_bfloat16* out_q;
  __nv_bfloat16* pool;
  const uint64_t* kv_off;   // element offset of row r's K slot within layer `layer`
  uint64_t layer_base;      // element offset of the layer plane
  uint32_t d;               // hidden width (Proj: N = 4d)
  uint32_t kv_stride;       // V offset from K = page_size * d
};

void launch_gemm(const GemmArgs& a, cudaStream_t s);
void launch_embed(__nv_bfloat16* x, const __nv_bfloat16* table, const uint32_t* tok, int rows, int d,
                  cudaStream_t s);

struct AttnArgs {
  const __nv_bfloat16* q;   // [rows x d]
  const __nv_bfloat16* pool;
  const uint32_t* pages;
  const ReqDev* reqs;
  const AttnItem* items;
  uint32_t n_items;
  float* part_o;            // [part_rows x d]
  float* part_lse;          // [part_rows x H]
  PoolGeom g;
  uint32_t layer;
  float scale_log2;         // log2(e) / sqrt(D)
  uint32_t bq;              // query rows per tile: 64 or 128 (items enumerate tiles of bq)
  unsigned long long* trace;  // optional per-CTA event timestamps (MTKV_ATTN_TRACE), else null
};
constexpr int kTraceCtas = 64, kTraceTiles = 32, kTraceKinds = 6;
void launch_attention(const AttnArgs& a, cudaStream_t s);

struct GateArgs {  // split combine + silu(o) * u + layer norm -> bf16
  const float* part_o;
  const float* part_lse;
  const __nv_bfloat16* u;
  const float* ln_scale;
  const uint32_t* row_req;
  const ReqDev* reqs;
  __nv_bfloat16* out;
  uint32_t rows, H, D;
};
void launch_gate_norm(const GateArgs& a, cudaStream_t s);

void launch_scatter_chunks(__nv_bfloat16* pool, const __nv_bfloat16* staging, const ChunkWork* work,
                           const uint32_t* pages, uint32_t n_chunks, const PoolGeom& g, cudaStream_t s);
void launch_gather_chunks(__nv_bfloat16* staging, const __nv_bfloat16* pool, const ChunkWork* work,
                          const uint32_t* pages, uint32_t n_chunks, const PoolGeom& g, cudaStream_t s);

// Tag backend: write identity patterns for every fresh history row, all layers.
void launch_tag_append(__nv_bfloat16* pool, const ReqDev* reqs, const uint32_t* pages, uint32_t n_reqs,
                       uint32_t max_hist, const PoolGeom& g, cudaStream_t s);

// Tag pattern of one 16-bit word (shared with the host checker).
__host__ __device__ inline uint16_t tag_word(uint32_t user, uint64_t pos, uint32_t layer, uint32_t kv,
                                             uint32_t j) {
  uint64_t t = ((uint64_t)user << 40) | ((pos & 0xFFFFFFFFull) << 8) | (layer & 0xFF);
  uint64_t x = t ^ ((uint64_t)kv << 63) ^ ((uint64_t)j * 0x9E3779B97F4A7C15ull);
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return (uint16_t)(x & 0xFFFF);
}

}  // namespace mtkv_b200

// ---- tcgen05 attention (attn_tc.cu): head_dim 64/128, page sizes 8..128 ----
#include <cuda.h>
namespace mtkv_b200 {
bool attn_tc_supported(const PoolGeom& g);
int make_pool_map(CUtensorMap* map, const void* pool, const PoolGeom& g);
void launch_attention_tc(const CUtensorMap& map, const AttnArgs& a, cudaStream_t s);
}  // namespace mtkv_b200
