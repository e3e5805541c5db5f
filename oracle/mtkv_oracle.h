/*
 * mtkv_oracle — CPU restatement (plain C11) of the reference's hierarchical
 * user-KV-cache serving path. TEST INFRASTRUCTURE ONLY: it is the checker the
 * parity tests, __graft_entry__.smoke() and bench.py's cpu_baseline leg call;
 * the product (paper_2604_22881_b200/) never links, loads or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks every output below against
 * (a) the known answers in the reference's own tests (tests/test_*.cpp,
 *     tests/acceptance.cpp) and
 * (b) golden fixtures produced by the UNMODIFIED reference compiled in place
 *     (oracle/_ref, tools/make_golden.py): full control-plane state after
 *     every batch (lengths, locks, recency stamps, page ids, counters, LRU
 *     order) and value-backend logits, bit-for-bit.
 *
 * Reference map (all paths under /root/reference/proj/core):
 *   orc_model_random      <- src/model.cpp:34  ModelParams::random
 *   orc_forward           <- src/model.cpp:140 forward_incremental (+ :104 attention,
 *                            :70 matmul, :86 layer_norm)
 *   LRU / manager         <- src/manager.cpp:7-229 LruIndex, CacheManager
 *   schedule              <- src/pipeline.cpp:25-95 Pipeline
 *   orc_engine_*          <- include/mtkv/sim.hpp:211-455 Engine<B>
 */
#ifndef MTKV_ORACLE_H
#define MTKV_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint32_t num_layers, num_heads, head_dim, page_size, chunk_size;
  uint32_t device_pages, onload_pages, bytes_per_element;
  uint64_t offload_quota, host_capacity;
} orc_kv_config;

typedef struct {
  double bus_bandwidth, tx_setup, host_bandwidth, page_op, attn_coeff;
  double linear_coeff, embed_coeff, layout_coeff;
  double meta_fixed, strip_fixed, embed_fixed, layout_fixed, await_fixed;
  double update_fixed, commit_per_chunk, offload_submit, post_fixed;
} orc_cost;

/* Model weights, row-major like the reference (model.hpp:32). */
typedef struct {
  uint32_t num_layers, num_heads, head_dim, vocab;
  const double* embed;  /* [vocab x d] */
  const double* w_in;   /* [L][d x 4d] */
  const double* ln;     /* [L][d] */
  const double* w1;     /* [L][d x d] */
  const double* w2;     /* [L][d x d] */
  const double* w_out;  /* [d x vocab] */
} orc_model;

enum { ORC_RECOMPUTE = 0, ORC_GPU_ONLY = 1, ORC_HIERARCHICAL = 2 };
enum { ORC_OK = 0, ORC_ERROR = 1, ORC_REJECTED = 2 };

typedef struct {
  uint32_t user;
  uint64_t history_len, reusable_len, device_served, host_onload, fresh_history;
  uint32_t delta, num_candidates, onload_chunks, scratch_pages;
} orc_plan;

typedef struct {
  uint32_t user;
  uint64_t freed_pages, tail_tokens_lost;
} orc_eviction;

typedef struct {
  uint64_t total_len, device_len, persisted_len, last_access;
  uint32_t locked, num_pages, host_chunks, pending_offload;
} orc_user_state;

typedef struct {
  double step_ms[9];
  double wait_ms, comp_ms, gpu_hit_ratio, total_hit_ratio;
  uint64_t tokens_processed, evictions, tail_tokens_lost, requests, batches;
  double avg_latency_ms, total_latency_ms;
  uint64_t peak_pages;
  uint64_t pages_allocated, occupied_pages, free_pages, quota_in_flight;
  double clock;
} orc_report;

typedef struct orc_engine orc_engine;

/* Defaults identical to the reference structs (core.hpp:29, costs.hpp:11). */
void orc_default_kv(orc_kv_config* c);
void orc_default_cost(orc_cost* c);

/* Weight init with the reference's RNG stream: mt19937_64 seeded with `seed`,
 * N(0, 0.3/sqrt(d)) via libstdc++'s polar normal_distribution, one fresh
 * distribution object per matrix, ln_scale ~ N(0,1). Buffers sized as above. */
void orc_model_random(uint32_t L, uint32_t H, uint32_t D, uint32_t vocab, uint64_t seed,
                      double* embed, double* w_in, double* ln, double* w1, double* w2,
                      double* w_out);

/* forward_incremental: cached_k/v are [L][cached_len][d]; fresh = delta ++ cands.
 * Writes logits [vocab]; new_k/new_v (nullable) get [L][M][d]. Returns ORC_OK or
 * ORC_ERROR (token out of vocabulary, no candidates). */
int orc_forward(const orc_model* m, const double* cached_k, const double* cached_v,
                uint64_t cached_len, const uint32_t* delta, uint32_t n_delta,
                const uint32_t* cands, uint32_t n_cands, double* logits,
                double* new_k, double* new_v);

/* Engine over a trace, batch by batch (sim.hpp:110). value_backend needs model. */
orc_engine* orc_engine_new(const orc_kv_config* kv, const orc_cost* cost, int mode,
                           uint32_t batch_size, int value_backend, const orc_model* model);
void orc_engine_free(orc_engine* e);
/* tokens: concatenated new tokens (value backend; may be NULL for tag);
 * cands: concatenated candidate ids (value backend). */
int orc_process_batch(orc_engine* e, uint32_t n, const uint64_t* ts, const uint32_t* users,
                      const uint32_t* dn, const uint32_t* nc, const uint32_t* tokens,
                      const uint32_t* cands);
void orc_drain(orc_engine* e);
const char* orc_last_error(const orc_engine* e);

uint32_t orc_last_plans(const orc_engine* e, orc_plan* out, uint32_t cap);
uint32_t orc_last_evictions(const orc_engine* e, orc_eviction* out, uint32_t cap);
uint32_t orc_last_logits(const orc_engine* e, double* out, uint32_t cap_rows); /* rows x vocab */
uint32_t orc_known_users(const orc_engine* e, uint32_t* out, uint32_t cap);    /* sorted */
int orc_user_state_get(const orc_engine* e, uint32_t user, orc_user_state* out);
uint32_t orc_user_pages(const orc_engine* e, uint32_t user, uint32_t* out, uint32_t cap);
uint32_t orc_lru_snapshot(const orc_engine* e, uint32_t* out, uint32_t cap); /* most recent first */
void orc_report_get(const orc_engine* e, orc_report* out);
/* Direct manager operations used by the safety/interleaving tests. */
int orc_evict_user(orc_engine* e, uint32_t user);
int orc_is_locked(const orc_engine* e, uint32_t user);

#ifdef __cplusplus
}
#endif
#endif
