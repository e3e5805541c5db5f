// Device-side data structures shared by the executor and the kernels.
//
// HBM layout of the paged store (paper §4.1, reference store.hpp:54):
//   pool[L][num_pages][2 (K,V)][page_size][H*D] bf16
// A page id addresses the same slot in every layer plane. Host chunks and the
// onload staging slots use [L][2][chunk_size][H*D] bf16, so one chunk is one
// contiguous copy-engine transfer.
#pragma once

#include <atomic>
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
  uint32_t seg0;        // first attention segment of this request (head-major, then query tile)
  uint32_t qtiles;      // query tiles of `bm` rows per head
  uint32_t split_keys;  // mma.sync path: keys per split
  uint32_t user;
  uint64_t dep_start;   // keys >= dep_start may be appended by this batch's projection GEMM
                        // (the user's first occurrence in the batch; later occurrences read them)
  uint32_t q_skip = 0;  // tcgen05 path: query rows [0, q_skip) are not computed (the last layer
                        // needs only each request's last row: model.cpp:195 reads e[last])
};

// Attention work decomposition. A segment = (request, head, query tile of bm
// rows) is one softmax problem; its partial results live in slots
// part_base .. part_base + n_parts - 1, each slot = bm rows x D floats (O / l)
// plus bm floats (log-sum-exp, base 2; -inf = empty). The split-K combine in
// gate_norm_kernel merges a segment's slots.
struct AttnSeg {
  uint32_t req, head, qtile;
  uint32_t n_tiles;     // tcgen05 path: 128-key tiles visible to the query tile
  uint32_t part_base, n_parts;
};
// tcgen05 path: a piece = key tiles [lo, hi) of one segment, run by one CTA of
// the persistent kernel; its partial result goes to slot `part`. The segment's
// and request's fields the kernel needs are copied in (one load per piece
// instead of a piece -> segment -> request chain of dependent loads).
struct alignas(16) AttnPiece {
  uint32_t seg, lo, hi, part;
  uint32_t head, qtile, q_row0, n_q;      // segment / request
  uint32_t n_hist, n_cand, pages_off, scratch_off;
  uint32_t n_scratch, q_skip;            // q_skip: the tile's rows are q_skip + qtile * bm + r
  uint32_t part_b = 0xFFFFFFFFu;         // paired kernel (attn_pair.cu): query tile qtile + 1's slot, or kNoPart
  uint32_t na = 0xFFFFFFFFu;             // paired kernel: tile qtile attends key tiles < na only
  uint64_t start, dep_start;
};
struct AttnItem {  // mma.sync path: one CTA = (request, head, query tile, key split)
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
  bool pdl = false;         // launch with programmatic stream serialization (the kernel
                            // waits for its predecessor before touching global data)
};

void launch_gemm(const GemmArgs& a, cudaStream_t s);
// tcgen05 path (gemm_tc.cu): Proj / SiluBf16 / Bf16 epilogues, K and N multiples of 64
bool gemm_tc_supported(const GemmArgs& a);
int launch_gemm_tc(const GemmArgs& a, uint64_t a_rows_alloc, cudaStream_t s);
void launch_embed(__nv_bfloat16* x, const __nv_bfloat16* table, const uint32_t* tok, int rows, int d,
                  cudaStream_t s);

// Partial-O slot layout (attention -> combine): per slot, 4-column chunks of
// all bm rows are contiguous ([slot][D/4 chunks][bm rows][4]). Thread r of the
// tcgen05 epilogue owns query row r, so a warp's 16-B stores of one chunk are
// 32 consecutive rows = 512 contiguous bytes (row-major slots made every
// store instruction touch 32 rows).
__host__ __device__ inline uint32_t part_chunks(uint32_t D) { return (D + 3) / 4; }
__host__ __device__ inline size_t part_index(uint32_t slot, uint32_t bm, uint32_t ri, uint32_t c, uint32_t D) {
  return ((size_t(slot) * part_chunks(D) + c / 4) * bm + ri) * 4 + (c & 3);
}
__host__ __device__ inline size_t part_slot_floats(uint32_t bm, uint32_t D) { return size_t(part_chunks(D)) * 4 * bm; }

constexpr uint32_t kNoPart = 0xFFFFFFFFu;

struct AttnArgs {
  const __nv_bfloat16* q;   // [rows x d]
  const __nv_bfloat16* pool;
  const uint32_t* pages;
  const ReqDev* reqs;
  const AttnSeg* segs;
  const AttnItem* items;    // mma.sync path: one per CTA
  uint32_t n_items;         // mma.sync path: CTAs; tcgen05 path: persistent CTAs
  const AttnPiece* pieces;  // tcgen05 path: pieces of CTA c = [cta_off[c], cta_off[c+1])
  const uint32_t* cta_off;
  float* part_o;            // [slots][D/4][bm][4] (part_index)
  float* part_lse;          // [slots x bm]
  PoolGeom g;
  uint32_t layer;
  float scale_log2;         // log2(e) / sqrt(D)
  uint32_t bq;              // query rows per tile: 64 or 128 (items enumerate tiles of bq)
  unsigned long long* trace;  // optional per-CTA event timestamps (MTKV_ATTN_TRACE), else null
  uint32_t trigger = 1;       // tcgen05 path: release the PDL dependent (gate_norm) at CTA start
  uint32_t pair = 0;          // tcgen05 path: the plan pairs query tiles (attn_pair_kernel)
};
constexpr int kTraceCtas = 64, kTraceTiles = 96, kTraceKinds = 12;
void launch_attention(const AttnArgs& a, cudaStream_t s);

struct GateArgs {  // split combine + silu(o) * u + layer norm -> bf16 (launched with PDL)
  const float* part_o;
  const float* part_lse;
  const AttnSeg* segs;
  uint32_t bm;              // query rows per segment (slot row stride)
  const __nv_bfloat16* u;
  const float* ln_scale;
  const uint32_t* row_req;
  const ReqDev* reqs;
  __nv_bfloat16* out;
  uint32_t rows, H, D;
  // row blocks (gate_block_kernel): (request, first query index) pairs, 32
  // query rows of one request each, aligned to the bm-row query tiles
  const uint32_t* blocks = nullptr;
  uint32_t n_blocks = 0;
  // optional: batch row of the gate operand u for output row `row` (the compact
  // last layer: out row r <- request r's last row)
  const uint32_t* u_rows = nullptr;
};
constexpr uint32_t kGateBlockRows = 32;
bool gate_block_supported(uint32_t H, uint32_t D);
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
int make_q_map(CUtensorMap* map, const void* q, uint64_t rows, const PoolGeom& g);
void launch_attention_tc(const CUtensorMap& pool_map, const CUtensorMap& q_map,
                         const AttnArgs& a, cudaStream_t s);
// two-lane form (attn_pp.cu): head_dim 64/128; planned over 2 x SMs virtual CTAs
// (an even count: CTA b runs virtual CTAs 2b and 2b + 1)
bool attn_pp_supported(const PoolGeom& g);
void launch_attention_pp(const CUtensorMap& pool_map, const CUtensorMap& q_map, const AttnArgs& a, cudaStream_t s);
// which attention kernel serves geometry g (attn_pp.cu: MTKV_ATTN=pp|mma select
// the two-lane or the mma.sync kernel for A/B measurements), and the virtual
// CTAs to plan for
enum class AttnKind { Mma, Tc, Pp };
AttnKind attn_kind(const PoolGeom& g);
uint32_t attn_plan_ctas(AttnKind k, int n_sm);
void launch_attention_any(AttnKind k, const CUtensorMap& pool_map, const CUtensorMap& q_map, const AttnArgs& a,
                          cudaStream_t s);
int num_sms();

// once per CUDA device (kernel attributes such as the dynamic smem opt-in are
// per device; a process may drive several GPUs)
struct DeviceOnce {
  static constexpr int kMaxDev = 64;
  std::atomic<bool> done[kMaxDev] = {};
  bool first() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev) return true;
    return !done[dev].exchange(true);
  }
};
}  // namespace mtkv_b200

// ---- host-side attention planning (attn_plan.cpp) ----
#include <vector>
namespace mtkv_b200 {
struct AttnPlan {
  uint32_t bm = 128;               // query rows per segment
  std::vector<AttnSeg> segs;
  std::vector<AttnPiece> pieces;   // tcgen05 path
  std::vector<uint32_t> cta_off;   // tcgen05 path, n_ctas + 1 entries
  std::vector<AttnItem> items;     // mma.sync path
  uint32_t n_slots = 0;
  bool pair = false;               // pieces are query-tile pairs (attn_pair_kernel)
  uint32_t n_ctas() const { return cta_off.empty() ? 0 : uint32_t(cta_off.size() - 1); }
};
constexpr uint32_t kTcBM = 128, kTcBN = 128;
// Fills reqs[r].seg0/qtiles (and split_keys for the mma path) and the plan.
// tcgen05: balanced contiguous key-tile ranges over `ctas` persistent CTAs.
// pair: units of two query tiles (2j, 2j+1) of one (request, head) share their
// key tiles (attn_pair_kernel, head_dim 128); a lone tile is a unit without B.
void plan_attention(ReqDev* reqs, uint32_t n, const PoolGeom& g, bool tc, uint32_t ctas, AttnPlan& plan,
                    bool pair = false);
// the batch has a request with more than one query tile and the paired kernel applies
bool attn_pair_wanted(const PoolGeom& g, const ReqDev* reqs, uint32_t n);
void launch_attention_pair(const CUtensorMap& pool_map, const CUtensorMap& q_map, const AttnArgs& a,
                           cudaStream_t s);
}  // namespace mtkv_b200
