/*
 * mtkv_b200.h — C-ABI of the B200-native hierarchical user-KV-cache serving path.
 *
 * Drop-in boundary for the reference's C++ serving API (namespace mtkv,
 * /root/reference/proj/core/include/mtkv/). Every entry point below names the
 * reference interface it replaces (file:line). Plain pointers and sizes only;
 * no torch or C++ types cross this boundary. Library: libmtkv_b200.so
 * (paper_2604_22881_b200/), built for sm_100a.
 *
 * Error behaviour mirrors the reference: where the reference throws
 * mtkv::Error a call returns MTKV_ERROR, where it throws mtkv::BatchRejected
 * it returns MTKV_BATCH_REJECTED; the message is available from
 * mtkv_last_error() (thread-local). Engine calls that need the GPU return
 * MTKV_NO_DEVICE when no CUDA device is usable — there is no CPU fallback.
 */
#ifndef MTKV_B200_H
#define MTKV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MTKV_OK 0
#define MTKV_ERROR 1
#define MTKV_BATCH_REJECTED 2
#define MTKV_NO_DEVICE 3

#define MTKV_MODE_RECOMPUTE 0    /* sim.hpp:25 Mode::Recompute */
#define MTKV_MODE_GPU_ONLY 1     /* Mode::GpuOnly */
#define MTKV_MODE_HIERARCHICAL 2 /* Mode::Hierarchical */

#define MTKV_BACKEND_TAG 0   /* store.hpp:19 TagBackend: payload = token identity */
#define MTKV_BACKEND_VALUE 1 /* store.hpp:38 ValueBackend: payload = model K/V */

/* core.hpp:29 KVConfig */
typedef struct {
  uint32_t num_layers, num_heads, head_dim, page_size, chunk_size;
  uint32_t device_pages, onload_pages, bytes_per_element;
  uint64_t offload_quota, host_capacity;
} mtkv_kv_config;

/* costs.hpp:11 CostModel (drives the deterministic event schedule) */
typedef struct {
  double bus_bandwidth, tx_setup, host_bandwidth, page_op, attn_coeff;
  double linear_coeff, embed_coeff, layout_coeff;
  double meta_fixed, strip_fixed, embed_fixed, layout_fixed, await_fixed;
  double update_fixed, commit_per_chunk, offload_submit, post_fixed;
} mtkv_cost_model;

/* model.hpp:12 ModelConfig */
typedef struct {
  uint32_t num_layers, num_heads, head_dim, vocab;
  uint64_t seed;
} mtkv_model_config;

/* core.hpp:58 Request. new_tokens / candidates may be NULL in tag mode
 * (counts only), as in the reference. */
typedef struct {
  uint64_t timestamp;
  uint32_t user;
  uint32_t new_token_count;
  uint32_t candidate_count;
  const uint32_t* new_tokens;
  const uint32_t* candidates;
} mtkv_request;

/* manager.hpp:51 RequestPlan (+ counts of its vectors) */
typedef struct {
  uint32_t user;
  uint64_t history_len, reusable_len, device_served, host_onload, fresh_history;
  uint32_t delta, num_candidates, onload_chunks, scratch_pages;
} mtkv_request_plan;

/* manager.hpp:44 EvictionRecord */
typedef struct {
  uint32_t user;
  uint64_t freed_pages, tail_tokens_lost;
} mtkv_eviction;

/* core.hpp:78 SequenceState (+ page/host/pending counts) */
typedef struct {
  uint64_t total_len, device_len, persisted_len, last_access;
  uint32_t locked, num_pages, host_chunks, pending_offload;
} mtkv_sequence_state;

/* sim.hpp:41 RunReport (+ control-plane counters and measured GPU timings) */
typedef struct {
  double step_ms[9];
  double wait_ms, comp_ms, gpu_hit_ratio, total_hit_ratio;
  uint64_t tokens_processed, evictions, tail_tokens_lost, requests, batches;
  double avg_latency_ms, total_latency_ms;
  uint64_t peak_pages;
  uint64_t pages_allocated, occupied_pages, free_pages, quota_in_flight;
  double clock;
  /* measured on the device (0 for a planner without executor) */
  uint64_t h2d_bytes, d2h_bytes, onload_chunks, offload_chunks;
  /* raw hit accounting behind the ratios (sim.hpp:70 HitAccumulator) */
  uint64_t hist_required, hist_device, hist_host;
  /* executor: host-hit prefix tokens brought back over the host link vs re-encoded on the SMs
     (onload_policy adaptive; the control plane counts both as host hits) */
  uint64_t prefix_onloaded, prefix_recomputed;
} mtkv_run_report;

typedef struct {
  int mode;              /* MTKV_MODE_* */
  int backend;           /* MTKV_BACKEND_* */
  uint32_t batch_size;   /* used by mtkv_engine_run (batchify) */
  uint64_t seed;
  mtkv_model_config model;  /* value backend */
  int device;               /* CUDA ordinal */
  uint32_t max_batch_tokens; /* fresh rows per batch the workspaces are sized for (0 = 65536) */
  uint32_t max_user_pages;   /* 0 = device_pages */
  uint32_t keep_logits;      /* 1: keep full [n x vocab] logits of the last batch */
  uint32_t profile;          /* 1: time every attention launch with CUDA events */
  uint64_t host_reserve_mb;  /* pinned host store allocated up front (0: grow on demand) */
  uint32_t device_planner;   /* 1: user lookup, LRU update, victim selection and page allocation
                                (manager.cpp:74 prepare_metadata) run on the GPU over device tables */
  uint32_t max_users;        /* device planner: user-table capacity (0 = 65536) */
  uint32_t host_extent_mb;   /* pinned host tier: per-user extent size (0 = 8 MB); an onload is one
                                copy-engine transfer per extent, so extents sized to a user's
                                persisted prefix keep the host link at its large-copy peak */
  uint32_t onload_policy;    /* 0 (MTKV_ONLOAD_ALWAYS): every host hit is onloaded over the host link,
                                as the reference executes it. 1 (MTKV_ONLOAD_ADAPTIVE): per batch, some
                                host-hit prefixes are re-encoded on the SMs instead, concurrently with the
                                onloads of the others, balancing estimated link time against recompute
                                time. Every control-plane decision, the simulated clock and the reported
                                hit ratios are unchanged (bit-exact); only how the prefix K/V reaches its
                                pages differs (bf16 recompute vs the stored bf16 bytes: numerics within the
                                engine's stated tolerance; tag backend: identical bytes). */
  double onload_gbs;         /* adaptive policy: host-link GB/s (0 = 54) */
  double recompute_mtok_s;   /* adaptive policy: prefix re-encode rate, M tokens/s (0 = from model dims) */
} mtkv_engine_options;
#define MTKV_ONLOAD_ALWAYS 0
#define MTKV_ONLOAD_ADAPTIVE 1

/* ---- configuration (core.cpp) ---- */
void mtkv_kv_config_default(mtkv_kv_config* out);                 /* core.hpp:29 defaults */
int mtkv_kv_config_validate(const mtkv_kv_config* c);             /* core.cpp:8 validate */
int mtkv_parse_config_text(const char* text, const char* origin,  /* core.cpp:28 */
                           mtkv_kv_config* out);
void mtkv_cost_model_default(mtkv_cost_model* out);               /* costs.hpp:11 */
uint64_t mtkv_pages_needed(uint64_t len, uint32_t page_size);     /* core.hpp:98 */
uint64_t mtkv_persisted_prefix(uint64_t len, uint32_t chunk_size);/* core.hpp:103 */
const char* mtkv_last_error(void);

/* ---- control plane: CacheManager + Pipeline schedule, host only ----
 * The planner is the half of Engine<B> that decides (manager.cpp:74
 * prepare_metadata, :141 evict_user, pipeline.cpp:25/78 schedule,
 * sim.hpp:212 process_due / :303 trigger_offloads). The engine runs the same
 * object ahead of the GPU; it is exposed so decisions can be replayed and
 * checked without a device. It computes no payloads. */
typedef struct mtkv_planner mtkv_planner;
mtkv_planner* mtkv_planner_create(const mtkv_kv_config* kv, const mtkv_cost_model* cost,
                                  int mode);
void mtkv_planner_destroy(mtkv_planner* p);
int mtkv_planner_process_batch(mtkv_planner* p, const mtkv_request* reqs, uint32_t n);
int mtkv_planner_drain(mtkv_planner* p);
/* The executor's host-hit policy as the planner applies it (mtkv_engine_options::
 * onload_policy, fixed rates: the engine measures them instead when given 0):
 * which host-hit prefix chunks a batch re-encodes and which it onloads (the
 * report's prefix_recomputed / prefix_onloaded). Control-plane decisions are
 * the same under every policy. */
int mtkv_planner_set_onload_policy(mtkv_planner* p, uint32_t policy, double onload_gbs, double recompute_mtok_s);
/* CacheManager step surface (manager.hpp:89-147) on the same host control
 * plane, for callers that drive the manager themselves the way
 * Engine<B>::process_batch does (sim.hpp:332-455). Request indices refer to the
 * last prepare; its plans / evictions are read with mtkv_last_plans /
 * mtkv_last_evictions (is_engine = 0). Errors carry the reference's messages. */
int mtkv_planner_prepare_metadata(mtkv_planner* p, const mtkv_request* reqs, uint32_t n,
                                  int host_enabled);                          /* manager.cpp:74 */
uint32_t mtkv_planner_scratch_pages(const mtkv_planner* p, uint32_t req, uint32_t* out,
                                    uint32_t cap);                            /* RequestPlan::scratch_pages */
/* release_scratch (manager.cpp:196): the plan's scratch page ids go back to the free list */
int mtkv_planner_release_scratch(mtkv_planner* p, const uint32_t* pages, uint32_t n);
/* commit_onload (manager.cpp:178): device_len = reusable_len when the plan onloaded chunks */
int mtkv_planner_commit_onload(mtkv_planner* p, uint32_t user, uint64_t reusable_len, uint32_t onload_chunks);
int mtkv_planner_finish_append(mtkv_planner* p, uint32_t user, uint64_t appended); /* :184 */
int mtkv_planner_advance_persisted(mtkv_planner* p, uint32_t user, uint64_t tokens); /* :190 */
int mtkv_planner_lock_user(mtkv_planner* p, uint32_t user);                  /* manager.cpp:165 */
int mtkv_planner_unlock_user(mtkv_planner* p, uint32_t user);                /* manager.cpp:172 */
uint32_t mtkv_planner_last_page_len(const mtkv_planner* p, uint32_t user);   /* manager.cpp:210 */

/* ---- engine: sim.hpp:110 Engine<B> on the GPU ---- */
typedef struct mtkv_engine mtkv_engine;
mtkv_engine* mtkv_engine_create(const mtkv_kv_config* kv, const mtkv_cost_model* cost,
                                const mtkv_engine_options* opts);
void mtkv_engine_destroy(mtkv_engine* e);
int mtkv_engine_process_batch(mtkv_engine* e, const mtkv_request* reqs, uint32_t n); /* sim.hpp:332 */
int mtkv_engine_run(mtkv_engine* e, const mtkv_request* trace, uint64_t n,           /* sim.hpp:135 */
                    mtkv_run_report* out);
int mtkv_engine_drain(mtkv_engine* e);                                              /* sim.hpp:145 */
int mtkv_engine_synchronize(mtkv_engine* e);
/* logit_sink (sim.hpp:104): logits of the last processed batch, rows x vocab fp32 */
int mtkv_engine_last_logits(mtkv_engine* e, float* out, uint32_t cap_rows);
/* rank_candidates (model.cpp:199) for each request of the last batch: writes
 * the candidate ids in descending logit order (stable) into out (concatenated) */
int mtkv_engine_last_rankings(mtkv_engine* e, uint32_t* out, uint64_t cap);
/* Pipelined serving: rankings of an earlier batch, identified by its ticket
 * (0-based index among successfully submitted batches), while later batches are
 * still in flight; the last 6 submitted batches stay readable. Blocks until that
 * batch has completed. The reference returns each batch's results from
 * Engine::process_batch (sim.hpp:332); this splits submit and read-back so the
 * host can enqueue batch i+1's onload before reading batch i. */
int mtkv_engine_batch_rankings(mtkv_engine* e, uint64_t ticket, uint32_t* out, uint64_t cap);
uint64_t mtkv_engine_batches_submitted(const mtkv_engine* e);
/* control-plane cost of the last batch: host wall ms of planning (prepare_metadata,
 * schedule, bookkeeping; includes the device planner's round trip when enabled)
 * and the device planner kernel's ms (0 with the host planner) */
void mtkv_engine_last_plan_ms(const mtkv_engine* e, double* plan_ms, double* ctl_kernel_ms);
/* check_conservation (sim.cpp:60), tag backend: reads back the whole device
 * pool and host store and verifies every resident token's identity */
int mtkv_engine_check_conservation(mtkv_engine* e);
/* reads one user's resident K/V of one layer in logical order (gather,
 * store.hpp:106) as raw bf16 bits: out_k/out_v hold cap_tokens x H*D */
int64_t mtkv_engine_read_user_kv(mtkv_engine* e, uint32_t user, uint32_t layer,
                                 uint16_t* out_k, uint16_t* out_v, uint64_t cap_tokens);
/* measured device time of the last batch (compute stream), milliseconds */
double mtkv_engine_last_batch_ms(mtkv_engine* e);
/* device time of the attention kernels of the last batch (ms) and their launch count */
double mtkv_engine_last_attention_ms(mtkv_engine* e, uint32_t* launches);
/* profile mode: device ms of the last batch's onload scatter (staging -> pages,
 * store.hpp:89) and offload gather (pages -> offload slots, store.hpp:106), with
 * the chunk counts they moved */
/* profile mode: device ms of the last batch's projection GEMMs, which append the
 * fresh rows' K/V into their pages (store.hpp:123 append), with launches and rows */
double mtkv_engine_last_proj_ms(mtkv_engine* e, uint32_t* launches, uint64_t* rows);
int mtkv_engine_last_chunk_copy_ms(mtkv_engine* e, double* scatter_ms, uint32_t* scatter_chunks,
                                   double* gather_ms, uint32_t* gather_chunks);
uint64_t mtkv_engine_kernel_launches(const mtkv_engine* e);
/* toggles per-launch CUDA-event timing of the attention kernels */
void mtkv_engine_set_profile(mtkv_engine* e, uint32_t on);
/* switches the executor's host-hit policy (mtkv_engine_options::onload_policy)
 * from the next batch on; the control plane is unaffected */
int mtkv_engine_set_onload_policy(mtkv_engine* e, uint32_t policy, double onload_gbs, double recompute_mtok_s);

/* ---- both objects: manager state (sim.hpp:149 manager()) ----
 * `obj` is an mtkv_planner* or mtkv_engine* as named by `is_engine`. */
int mtkv_report(const void* obj, int is_engine, mtkv_run_report* out);      /* sim.hpp:457 */
uint32_t mtkv_last_plans(const void* obj, int is_engine, mtkv_request_plan* out, uint32_t cap);
uint32_t mtkv_last_evictions(const void* obj, int is_engine, mtkv_eviction* out, uint32_t cap);
uint32_t mtkv_known_users(const void* obj, int is_engine, uint32_t* out, uint32_t cap); /* manager.hpp:131 */
int mtkv_user_state(const void* obj, int is_engine, uint32_t user, mtkv_sequence_state* out);
uint32_t mtkv_user_pages(const void* obj, int is_engine, uint32_t user, uint32_t* out, uint32_t cap); /* :125 */
uint32_t mtkv_lru_snapshot(const void* obj, int is_engine, uint32_t* out, uint32_t cap);  /* :37 */
int mtkv_evict_user(void* obj, int is_engine, uint32_t user);                /* manager.cpp:141 */
int mtkv_is_locked(const void* obj, int is_engine, uint32_t user);           /* manager.hpp:112 */
uint64_t mtkv_get_total_cache_length(const void* obj, int is_engine, uint32_t user); /* :96 */
/* Engine<B>::dump_page_map (sim.hpp:493): {"user":[page ids],...} over the known
 * users in id order, byte-identical to the reference's string. malloc'd, free
 * with mtkv_free. */
char* mtkv_dump_page_map(const void* obj, int is_engine);
/* Canonical binary image of the complete control-plane state (the fields of the
 * reference driver's state dump: oracle/ref_driver.cpp dump_state), for
 * bit-exact comparison at trace scale. Little-endian:
 *   "MTKVST01", u64 n_users, then per known user in id order
 *     u32 user, u32 locked, u64 total_len, device_len, persisted_len, last_access,
 *     host_chunks, pending_offload, n_pages, u32 pages[n_pages];
 *   u64 n_lru, u32 lru[n_lru] (most recent first);
 *   u64 evictions, tail_tokens_lost, pages_allocated, occupied_pages, free_pages,
 *     quota_in_flight; f64 clock.
 * Writes min(size, cap) bytes to buf (may be NULL) and returns the full size. */
int64_t mtkv_state_blob(const void* obj, int is_engine, uint8_t* buf, uint64_t cap);

/* ---- workload (workload.cpp): identical RNG streams to the reference ---- */
typedef struct {
  uint32_t num_users;
  uint64_t total_requests;
  int pareto;  /* TailFamily */
  double gap_log_mu, gap_log_sigma, pareto_alpha, pareto_scale_ms;
  double mean_final_len;
  uint64_t min_len, max_len;
  uint32_t fixed_delta, candidates, vocab;
  uint64_t seed;
} mtkv_gen_config;
void mtkv_gen_config_default(mtkv_gen_config* out);                  /* workload.hpp:15 */
int mtkv_gen_config_preset(const char* name, mtkv_gen_config* out);  /* workload.cpp:28-56 */
/* generate_trace (workload.cpp:85) into a JSONL string (the reference's trace
 * format, workload.cpp:182); returns malloc'd text, free with mtkv_free. */
char* mtkv_generate_trace_jsonl(const mtkv_gen_config* g);
void mtkv_free(void* p);

/* ---- raw device ops on caller-owned device pointers (kernel-level parity) ----
 * Paged pool layout: [L][num_pages][2][page_size][H*D] bf16. */
int mtkv_op_scatter_chunks(void* pool, const void* staging, const uint32_t* d_page_ids,
                           uint32_t n_chunks, const mtkv_kv_config* kv, uint32_t num_pages,
                           void* stream);
int mtkv_op_gather_chunks(void* staging, const void* pool, const uint32_t* d_page_ids,
                          uint32_t n_chunks, const mtkv_kv_config* kv, uint32_t num_pages,
                          void* stream);
/* Incremental prefix-reuse attention for one request and one layer: queries q
 * [n_q x H*D] bf16 at positions p_pre..p_pre+n_q-1 over keys of positions
 * 0..n_keys-1 held in the pages d_pages (first n_keys slots, in order);
 * out [n_q x H*D] fp32. */
int mtkv_op_paged_attention(float* out, const void* q, const void* pool, const uint32_t* d_pages,
                            uint32_t n_q, uint64_t p_pre, uint64_t n_keys, uint32_t layer,
                            const mtkv_kv_config* kv, uint32_t num_pages, void* stream);
/* Batched form: request r's fresh rows (q rows [sum n_q[<r], +n_q[r])) attend over
 * its p_pre[r] cached keys and themselves; its page ids start at
 * d_pages[page_off[r]] (host arrays page_off / n_q / p_pre). repeat > 1 launches
 * the attention kernel `repeat` times and returns the mean device ms of launches
 * 2..repeat in *ms_per_launch, each timed alone after an L2-evicting memset
 * (kernel benchmarking); out gets the merged result. */
int mtkv_op_paged_attention_batch(float* out, const void* q, const void* pool, const uint32_t* d_pages,
                                  const uint32_t* page_off, const uint32_t* n_q, const uint64_t* p_pre,
                                  uint32_t n_req, uint32_t layer, const mtkv_kv_config* kv, uint32_t num_pages,
                                  uint32_t repeat, float* ms_per_launch, void* stream);
/* Dense layer of the GR block (model.cpp:71 matmul; act = 1 applies the block's
 * silu, model.cpp:174/:191): out[M x N] bf16 = act(a[M x K] . w[K x N]) with bf16
 * operands (w row-major, the reference's layout) and fp32 accumulation, on the
 * tcgen05 kernel when K and N are multiples of 64 (tc = 1: refuse other shapes),
 * else the mma.sync kernel. a_rows_alloc = rows allocated behind `a` (>= M). */
int mtkv_op_dense(void* out, const void* a, const void* w, uint32_t M, uint32_t N, uint32_t K,
                  uint64_t a_rows_alloc, int act, int tc, void* stream);
/* Host-only self-check of the attention work planner (attn_plan.cpp): plans a
 * batch (fresh history rows, candidates and cached prefix per request) for
 * `ctas` persistent CTAs and verifies every (request, head, query tile, key
 * tile) is covered exactly once and partial slots are contiguous. Returns 0 or
 * a failure code; out_stats[5] = {segments, pieces, tiles, max tiles per CTA, CTAs}.
 * tc: 0 = mma.sync items, 1 = one query tile per piece (attn_tc_kernel),
 * 2 = paired query tiles (attn_pair_kernel; tiles counts key tiles streamed). */
int mtkv_attention_plan_check(uint32_t n, const uint32_t* n_hist, const uint32_t* n_cand, const uint64_t* start,
                              uint32_t H, uint32_t D, uint32_t S, uint32_t ctas, int tc, uint32_t* out_stats);

#ifdef __cplusplus
}
#endif
#endif /* MTKV_B200_H */
