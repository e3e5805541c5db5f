/*
 * mtkv_oracle.c — CPU restatement of the reference serving path. TEST
 * INFRASTRUCTURE ONLY (see mtkv_oracle.h for the contract and reference map).
 * Written as flat C: user table in an open-addressing hash, intrusive LRU
 * links, LIFO page stack, binary heap of pending offload completions.
 */
#include "mtkv_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ RNG --- */
/* mt19937_64 (same recurrence libstdc++ implements) */
typedef struct { uint64_t mt[312]; int idx; } mt64;

static void mt64_seed(mt64* r, uint64_t s) {
  r->mt[0] = s;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

static uint64_t mt64_next(mt64* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* libstdc++ generate_canonical<double,53> over a 64-bit engine: one draw / 2^64 */
static double canon01(mt64* r) {
  double v = (double)mt64_next(r) / 18446744073709551616.0;
  if (v >= 1.0) v = nextafter(1.0, 0.0);
  return v;
}

/* libstdc++ normal_distribution (Marsaglia polar, caches the second variate) */
typedef struct { int saved_ok; double saved; } normal_state;

static double normal_draw(normal_state* st, mt64* r, double mean, double sd) {
  double ret;
  if (st->saved_ok) {
    st->saved_ok = 0;
    ret = st->saved;
  } else {
    double x, y, r2;
    do {
      x = 2.0 * canon01(r) - 1.0;
      y = 2.0 * canon01(r) - 1.0;
      r2 = x * x + y * y;
    } while (r2 > 1.0 || r2 == 0.0);
    double mult = sqrt(-2 * log(r2) / r2);
    st->saved = x * mult;
    st->saved_ok = 1;
    ret = y * mult;
  }
  return ret * sd + mean;
}

static void fill_normal(mt64* r, double* out, size_t n, double sd) {
  normal_state st = {0, 0.0};
  for (size_t i = 0; i < n; ++i) out[i] = normal_draw(&st, r, 0.0, sd);
}

void orc_model_random(uint32_t L, uint32_t H, uint32_t D, uint32_t vocab, uint64_t seed,
                      double* embed, double* w_in, double* ln, double* w1, double* w2,
                      double* w_out) {
  mt64 r;
  mt64_seed(&r, seed);
  size_t d = (size_t)H * D;
  double s = 0.3 / sqrt((double)d);
  fill_normal(&r, embed, (size_t)vocab * d, s);
  for (uint32_t l = 0; l < L; ++l) {
    fill_normal(&r, w_in + (size_t)l * d * 4 * d, d * 4 * d, s);
    fill_normal(&r, ln + (size_t)l * d, d, 1.0);
    fill_normal(&r, w1 + (size_t)l * d * d, d * d, s);
    fill_normal(&r, w2 + (size_t)l * d * d, d * d, s);
  }
  fill_normal(&r, w_out, d * vocab, s);
}

/* ---------------------------------------------------------------- model --- */
static double silu(double x) { return x / (1.0 + exp(-x)); }

/* y[rows x n] = x[rows x m] @ w[m x n]; zero inputs skipped like the reference */
static void mm(const double* x, const double* w, double* y, size_t rows, size_t m, size_t n) {
  for (size_t r = 0; r < rows; ++r) {
    double* yr = y + r * n;
    for (size_t j = 0; j < n; ++j) yr[j] = 0.0;
    const double* xr = x + r * m;
    for (size_t k = 0; k < m; ++k) {
      double xv = xr[k];
      if (xv == 0.0) continue;
      const double* wk = w + k * n;
      for (size_t j = 0; j < n; ++j) yr[j] += xv * wk[j];
    }
  }
}

static void norm_rows(double* x, const double* scale, size_t rows, size_t d) {
  for (size_t r = 0; r < rows; ++r) {
    double* row = x + r * d;
    double mean = 0.0;
    for (size_t j = 0; j < d; ++j) mean += row[j];
    mean /= (double)d;
    double var = 0.0;
    for (size_t j = 0; j < d; ++j) {
      double c = row[j] - mean;
      var += c * c;
    }
    var /= (double)d;
    double inv = 1.0 / sqrt(var + 1e-6);
    for (size_t j = 0; j < d; ++j) row[j] = (row[j] - mean) * inv * scale[j];
  }
}

int orc_forward(const orc_model* m, const double* ck, const double* cv, uint64_t clen,
                const uint32_t* delta, uint32_t nd, const uint32_t* cands, uint32_t nc,
                double* logits, double* new_k, double* new_v) {
  if (nc == 0) return ORC_ERROR;
  const size_t d = (size_t)m->num_heads * m->head_dim, M = (size_t)nd + nc;
  const size_t H = m->num_heads, Dh = m->head_dim;
  for (size_t i = 0; i < M; ++i) {
    uint32_t t = i < nd ? delta[i] : cands[i - nd];
    if (t >= m->vocab) return ORC_ERROR;
  }
  double* e = malloc(M * d * sizeof(double));
  double* proj = malloc(M * 4 * d * sizeof(double));
  double* u = malloc(M * d * sizeof(double));
  double* q = malloc(M * d * sizeof(double));
  double* k = malloc(M * d * sizeof(double));
  double* v = malloc(M * d * sizeof(double));
  double* att = malloc(M * d * sizeof(double));
  double* mid = malloc(M * d * sizeof(double));
  double* sc = malloc((clen + M + 1) * sizeof(double));
  for (size_t i = 0; i < M; ++i) {
    uint32_t t = i < nd ? delta[i] : cands[i - nd];
    memcpy(e + i * d, m->embed + (size_t)t * d, d * sizeof(double));
  }
  const double scale = 1.0 / sqrt((double)Dh);
  for (uint32_t l = 0; l < m->num_layers; ++l) {
    mm(e, m->w_in + (size_t)l * d * 4 * d, proj, M, d, 4 * d);
    for (size_t i = 0; i < M * 4 * d; ++i) proj[i] = silu(proj[i]);
    for (size_t i = 0; i < M; ++i) {
      memcpy(u + i * d, proj + i * 4 * d, d * sizeof(double));
      memcpy(q + i * d, proj + i * 4 * d + d, d * sizeof(double));
      memcpy(k + i * d, proj + i * 4 * d + 2 * d, d * sizeof(double));
      memcpy(v + i * d, proj + i * 4 * d + 3 * d, d * sizeof(double));
    }
    const double* lk = ck ? ck + (size_t)l * clen * d : NULL;
    const double* lv = cv ? cv + (size_t)l * clen * d : NULL;
    for (size_t i = 0; i < M; ++i) {
      size_t span = clen + i + 1;
      for (size_t h = 0; h < H; ++h) {
        const double* qi = q + i * d + h * Dh;
        for (size_t j = 0; j < span; ++j) {
          const double* kj = j < clen ? lk + j * d + h * Dh : k + (j - clen) * d + h * Dh;
          double dot = 0.0;
          for (size_t t = 0; t < Dh; ++t) dot += qi[t] * kj[t];
          sc[j] = dot * scale;
        }
        double mx = sc[0];
        for (size_t j = 1; j < span; ++j)
          if (sc[j] > mx) mx = sc[j];
        double sum = 0.0;
        for (size_t j = 0; j < span; ++j) {
          sc[j] = exp(sc[j] - mx);
          sum += sc[j];
        }
        double* oi = att + i * d + h * Dh;
        for (size_t t = 0; t < Dh; ++t) oi[t] = 0.0;
        for (size_t j = 0; j < span; ++j) {
          double p = sc[j] / sum;
          const double* vj = j < clen ? lv + j * d + h * Dh : v + (j - clen) * d + h * Dh;
          for (size_t t = 0; t < Dh; ++t) oi[t] += p * vj[t];
        }
      }
    }
    if (new_k) memcpy(new_k + (size_t)l * M * d, k, M * d * sizeof(double));
    if (new_v) memcpy(new_v + (size_t)l * M * d, v, M * d * sizeof(double));
    for (size_t i = 0; i < M * d; ++i) att[i] = silu(att[i]) * u[i];
    norm_rows(att, m->ln + (size_t)l * d, M, d);
    mm(att, m->w1 + (size_t)l * d * d, mid, M, d, d);
    for (size_t i = 0; i < M * d; ++i) mid[i] = silu(mid[i]);
    mm(mid, m->w2 + (size_t)l * d * d, e, M, d, d);
  }
  mm(e + (M - 1) * d, m->w_out, logits, 1, d, m->vocab);
  free(e); free(proj); free(u); free(q); free(k); free(v); free(att); free(mid); free(sc);
  return ORC_OK;
}

/* ------------------------------------------------------------- helpers --- */
typedef struct { uint32_t* v; size_t n, cap; } u32vec;
static void u32_push(u32vec* a, uint32_t x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 16;
    a->v = realloc(a->v, a->cap * sizeof(uint32_t));
  }
  a->v[a->n++] = x;
}
typedef struct { double* v; size_t n, cap; } f64vec;
static void f64_reserve(f64vec* a, size_t n) {
  if (n > a->cap) {
    size_t c = a->cap ? a->cap : 64;
    while (c < n) c *= 2;
    a->v = realloc(a->v, c * sizeof(double));
    a->cap = c;
  }
}

typedef struct {
  uint32_t id;
  int known;                 /* present in the manager's sequence table */
  uint64_t total_len, device_len, persisted_len, last_access;
  int locked;
  int has_pages;             /* page-table entry exists */
  u32vec pages;
  int in_lru, prev, next;    /* LRU links (slots); prev = more recent */
  uint32_t host_chunks, pending;
  uint64_t recompute_len;
  u32vec hist;               /* value backend: full token history */
  f64vec kv;                 /* value backend: canonical K/V, [pos][L][2][d] */
  uint64_t kv_len;
} user_t;

typedef struct { double done; uint64_t order; uint32_t slot; uint64_t chunk; } pend_t;

struct orc_engine {
  orc_kv_config kv;
  orc_cost cost;
  int mode, value;
  uint32_t batch_size;
  orc_model model;
  /* users */
  user_t* users;
  size_t n_users, cap_users;
  int32_t* hslots;   /* hash table -> user slot, -1 empty */
  size_t hcap;
  /* LRU list */
  int lru_head, lru_tail;
  size_t lru_size;
  /* device page stack */
  uint32_t* stack;
  size_t stack_n;
  uint64_t occupied, clockc, evictions, tail_lost, pages_allocated;
  uint64_t host_total;
  /* schedule */
  double chunk_bytes, host_cpu_avail, onload_avail, scatter_avail, offload_avail, pinned_free[2];
  uint64_t pinned_next;
  pend_t* heap;
  size_t heap_n, heap_cap;
  uint64_t order;
  uint64_t quota_in_flight;
  /* report */
  double clock, step_sum[9], wait_sum, comp_sum, latency_sum;
  uint64_t required, dev_served, host_served, tokens_processed, requests, batches, peak_pages;
  /* last batch */
  orc_plan* plans;
  size_t n_plans, cap_plans;
  orc_eviction* evs;
  size_t n_evs, cap_evs;
  double* logits;
  size_t n_logit_rows;
  uint32_t* scratch;
  size_t n_scratch, cap_scratch;
  char err[256];
};

static uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

static int find_slot(const orc_engine* e, uint32_t id) {
  size_t m = e->hcap - 1, h = hash32(id) & m;
  while (e->hslots[h] >= 0) {
    if (e->users[e->hslots[h]].id == id) return e->hslots[h];
    h = (h + 1) & m;
  }
  return -1;
}

static void rehash(orc_engine* e) {
  size_t nc = e->hcap * 2;
  int32_t* ns = malloc(nc * sizeof(int32_t));
  for (size_t i = 0; i < nc; ++i) ns[i] = -1;
  for (size_t s = 0; s < e->n_users; ++s) {
    size_t h = hash32(e->users[s].id) & (nc - 1);
    while (ns[h] >= 0) h = (h + 1) & (nc - 1);
    ns[h] = (int32_t)s;
  }
  free(e->hslots);
  e->hslots = ns;
  e->hcap = nc;
}

static int get_slot(orc_engine* e, uint32_t id) {
  int s = find_slot(e, id);
  if (s >= 0) return s;
  if ((e->n_users + 1) * 2 > e->hcap) rehash(e);
  if (e->n_users == e->cap_users) {
    e->cap_users = e->cap_users ? 2 * e->cap_users : 64;
    e->users = realloc(e->users, e->cap_users * sizeof(user_t));
  }
  user_t* u = &e->users[e->n_users];
  memset(u, 0, sizeof(*u));
  u->id = id;
  u->prev = u->next = -1;
  size_t h = hash32(id) & (e->hcap - 1);
  while (e->hslots[h] >= 0) h = (h + 1) & (e->hcap - 1);
  e->hslots[h] = (int32_t)e->n_users;
  return (int)e->n_users++;
}

/* ---------------------------------------------------------------- LRU --- */
static void lru_unlink(orc_engine* e, int s) {
  user_t* u = &e->users[s];
  if (!u->in_lru) return;
  if (u->prev >= 0) e->users[u->prev].next = u->next; else e->lru_head = u->next;
  if (u->next >= 0) e->users[u->next].prev = u->prev; else e->lru_tail = u->prev;
  u->prev = u->next = -1;
  u->in_lru = 0;
  e->lru_size--;
}

static void lru_touch(orc_engine* e, int s) {
  lru_unlink(e, s);
  user_t* u = &e->users[s];
  u->next = e->lru_head;
  u->prev = -1;
  if (e->lru_head >= 0) e->users[e->lru_head].prev = s; else e->lru_tail = s;
  e->lru_head = s;
  u->in_lru = 1;
  e->lru_size++;
}

/* ------------------------------------------------------------ manager --- */
static uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

static uint32_t page_pop(orc_engine* e) {
  uint32_t p = e->stack[--e->stack_n];
  e->occupied++;
  e->pages_allocated++;
  return p;
}
static void page_push(orc_engine* e, uint32_t p) {
  e->stack[e->stack_n++] = p;
  e->occupied--;
}

static int evict(orc_engine* e, int s, uint64_t* freed) {
  user_t* u = &e->users[s];
  if (u->locked) { snprintf(e->err, sizeof e->err, "evict: user is locked"); return ORC_ERROR; }
  if (!u->known) { snprintf(e->err, sizeof e->err, "evict: unknown user"); return ORC_ERROR; }
  uint64_t n = 0;
  if (u->has_pages) {
    n = u->pages.n;
    for (size_t i = 0; i < u->pages.n; ++i) page_push(e, u->pages.v[i]);
    u->pages.n = 0;
    u->has_pages = 0;
  }
  if (u->device_len > u->persisted_len) e->tail_lost += u->device_len - u->persisted_len;
  u->device_len = 0;
  e->evictions++;
  lru_unlink(e, s);
  if (freed) *freed = n;
  return ORC_OK;
}

static void log_eviction(orc_engine* e, uint32_t user, uint64_t freed, uint64_t tail) {
  if (e->n_evs == e->cap_evs) {
    e->cap_evs = e->cap_evs ? 2 * e->cap_evs : 16;
    e->evs = realloc(e->evs, e->cap_evs * sizeof(orc_eviction));
  }
  e->evs[e->n_evs].user = user;
  e->evs[e->n_evs].freed_pages = freed;
  e->evs[e->n_evs].tail_tokens_lost = tail;
  e->n_evs++;
}

/* frees pages by evicting the least-recent users that are neither batch
 * members (`inbatch` mark) nor locked (manager.cpp:55 ensure_free) */
static int make_room(orc_engine* e, uint64_t needed, const unsigned char* inbatch) {
  while (e->stack_n < needed) {
    int v = e->lru_tail;
    while (v >= 0 && (inbatch[v] || e->users[v].locked)) v = e->users[v].prev;
    if (v < 0) {
      snprintf(e->err, sizeof e->err, "allocation unsatisfiable: all resident users locked or in batch");
      return ORC_REJECTED;
    }
    user_t* u = &e->users[v];
    uint64_t tail = u->device_len > u->persisted_len ? u->device_len - u->persisted_len : 0;
    uint64_t freed = 0;
    evict(e, v, &freed);
    log_eviction(e, u->id, freed, tail);
  }
  return ORC_OK;
}

/* --------------------------------------------------------- scheduling --- */
static void heap_push(orc_engine* e, pend_t p) {
  if (e->heap_n == e->heap_cap) {
    e->heap_cap = e->heap_cap ? 2 * e->heap_cap : 64;
    e->heap = realloc(e->heap, e->heap_cap * sizeof(pend_t));
  }
  size_t i = e->heap_n++;
  e->heap[i] = p;
  while (i > 0) {
    size_t par = (i - 1) / 2;
    pend_t* a = &e->heap[par];
    pend_t* b = &e->heap[i];
    if (a->done < b->done || (a->done == b->done && a->order < b->order)) break;
    pend_t t = *a; *a = *b; *b = t;
    i = par;
  }
}
static int heap_less(const pend_t* a, const pend_t* b) {
  return a->done < b->done || (a->done == b->done && a->order < b->order);
}
static pend_t heap_pop(orc_engine* e) {
  pend_t top = e->heap[0];
  e->heap[0] = e->heap[--e->heap_n];
  size_t i = 0;
  for (;;) {
    size_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < e->heap_n && heap_less(&e->heap[l], &e->heap[m])) m = l;
    if (r < e->heap_n && heap_less(&e->heap[r], &e->heap[m])) m = r;
    if (m == i) break;
    pend_t t = e->heap[m]; e->heap[m] = e->heap[i]; e->heap[i] = t;
    i = m;
  }
  return top;
}

/* sim.hpp:212 process_due */
static int complete_due(orc_engine* e, double now) {
  while (e->heap_n > 0 && e->heap[0].done <= now) {
    pend_t p = heap_pop(e);
    user_t* u = &e->users[p.slot];
    if (p.chunk != u->host_chunks) { snprintf(e->err, sizeof e->err, "host write: gap in chunk sequence"); return ORC_ERROR; }
    if (e->kv.host_capacity != 0 && e->host_total >= e->kv.host_capacity) {
      snprintf(e->err, sizeof e->err, "host write: capacity exceeded");
      return ORC_ERROR;
    }
    u->host_chunks++;
    e->host_total++;
    u->persisted_len += e->kv.chunk_size;
    if (u->persisted_len > u->total_len) { snprintf(e->err, sizeof e->err, "persist: beyond total length"); return ORC_ERROR; }
    e->quota_in_flight -= e->kv.chunk_size;
    if (--u->pending == 0) u->locked = 0;
  }
  return ORC_OK;
}

/* pipeline.cpp:25 submit_onload -> per-layer fire times */
static void schedule_onload(orc_engine* e, double submit, size_t n_chunks, double* fire) {
  const uint32_t L = e->kv.num_layers;
  for (uint32_t l = 0; l < L; ++l) fire[l] = submit;
  if (n_chunks == 0) return;
  const double fill = e->chunk_bytes / e->cost.host_bandwidth;
  const double dma = e->cost.tx_setup + e->chunk_bytes / e->cost.bus_bandwidth;
  const double scat = (double)(e->kv.chunk_size / e->kv.page_size) * e->cost.page_op;
  for (size_t c = 0; c < n_chunks; ++c) {
    uint64_t buf = e->pinned_next++ % 2;
    double fs = e->host_cpu_avail;
    if (e->pinned_free[buf] > fs) fs = e->pinned_free[buf];
    if (submit > fs) fs = submit;
    double fe = fs + fill;
    e->host_cpu_avail = fe;
    double ds = e->onload_avail > fe ? e->onload_avail : fe;
    double de = ds + dma;
    e->onload_avail = de;
    e->pinned_free[buf] = de;
    for (uint32_t l = 0; l < L; ++l) {
      double ss = e->scatter_avail > de ? e->scatter_avail : de;
      double se = ss + scat;
      e->scatter_avail = se;
      if (se > fire[l]) fire[l] = se;
    }
  }
  for (uint32_t l = 1; l < L; ++l)
    if (fire[l - 1] > fire[l]) fire[l] = fire[l - 1];
}

/* pipeline.cpp:78 submit_offload -> completion time */
static double schedule_offload(orc_engine* e, double submit) {
  const double gather = (double)e->kv.num_layers * (double)(e->kv.chunk_size / e->kv.page_size) * e->cost.page_op;
  const double dma = e->cost.tx_setup + e->chunk_bytes / e->cost.bus_bandwidth;
  const double copy = e->chunk_bytes / e->cost.host_bandwidth;
  double gs = e->offload_avail > submit ? e->offload_avail : submit;
  double ge = gs + gather;
  double de = ge + dma;
  e->offload_avail = de;
  return de + copy;
}

/* sim.hpp:303 trigger_offloads */
static void offload_ready_chunks(orc_engine* e, int s, double t) {
  user_t* u = &e->users[s];
  const uint64_t C = e->kv.chunk_size;
  for (;;) {
    uint64_t covered = u->persisted_len + (uint64_t)u->pending * C;
    if (u->device_len < covered + C) break;
    if (e->quota_in_flight + C > e->kv.offload_quota) break;
    e->quota_in_flight += C;
    double done = schedule_offload(e, t);
    if (u->pending == 0) u->locked = 1;
    u->pending++;
    pend_t p = {done, e->order++, (uint32_t)s, covered / C};
    heap_push(e, p);
  }
}

/* ------------------------------------------------------------- engine --- */
void orc_default_kv(orc_kv_config* c) {
  c->num_layers = 8; c->num_heads = 4; c->head_dim = 128; c->page_size = 32;
  c->chunk_size = 1024; c->device_pages = 40960; c->onload_pages = 10008;
  c->bytes_per_element = 2; c->offload_quota = 8192; c->host_capacity = 0;
}

void orc_default_cost(orc_cost* c) {
  c->bus_bandwidth = 25e9; c->tx_setup = 10e-6; c->host_bandwidth = 50e9; c->page_op = 50e-9;
  c->attn_coeff = 2e-10; c->linear_coeff = 1e-7; c->embed_coeff = 5e-8; c->layout_coeff = 5e-8;
  c->meta_fixed = 1e-4; c->strip_fixed = 5e-5; c->embed_fixed = 1e-4; c->layout_fixed = 1e-4;
  c->await_fixed = 5e-5; c->update_fixed = 5e-5; c->commit_per_chunk = 5e-6;
  c->offload_submit = 3e-5; c->post_fixed = 2e-4;
}

orc_engine* orc_engine_new(const orc_kv_config* kv, const orc_cost* cost, int mode,
                           uint32_t batch_size, int value_backend, const orc_model* model) {
  if (kv->page_size < 1 || kv->chunk_size < kv->page_size || kv->chunk_size % kv->page_size ||
      kv->device_pages < 1 || kv->offload_quota < kv->chunk_size || batch_size < 1)
    return NULL;
  if (value_backend && !model) return NULL;
  orc_engine* e = calloc(1, sizeof(orc_engine));
  e->kv = *kv;
  e->cost = *cost;
  e->mode = mode;
  e->value = value_backend;
  e->batch_size = batch_size;
  if (model) e->model = *model;
  e->hcap = 64;
  e->hslots = malloc(e->hcap * sizeof(int32_t));
  for (size_t i = 0; i < e->hcap; ++i) e->hslots[i] = -1;
  e->lru_head = e->lru_tail = -1;
  e->stack = malloc(kv->device_pages * sizeof(uint32_t));
  for (uint32_t i = 0; i < kv->device_pages; ++i) e->stack[i] = kv->device_pages - 1 - i;
  e->stack_n = kv->device_pages;
  uint64_t token_bytes = (uint64_t)kv->num_layers * 2 * kv->num_heads * kv->head_dim * kv->bytes_per_element;
  e->chunk_bytes = (double)kv->chunk_size * (double)token_bytes;
  return e;
}

void orc_engine_free(orc_engine* e) {
  if (!e) return;
  for (size_t s = 0; s < e->n_users; ++s) {
    free(e->users[s].pages.v);
    free(e->users[s].hist.v);
    free(e->users[s].kv.v);
  }
  free(e->users); free(e->hslots); free(e->stack); free(e->heap);
  free(e->plans); free(e->evs); free(e->logits); free(e->scratch);
  free(e);
}

const char* orc_last_error(const orc_engine* e) { return e->err; }

/* Value backend: run the model for one request and extend the canonical KV. */
static int encode_value(orc_engine* e, int s, const orc_plan* p, const uint32_t* newtok,
                        const uint32_t* cands, double* logits) {
  user_t* u = &e->users[s];
  const size_t L = e->kv.num_layers, d = (size_t)e->kv.num_heads * e->kv.head_dim;
  if (u->hist.n != p->history_len) {
    snprintf(e->err, sizeof e->err, "value mode: trace must carry explicit token ids");
    return ORC_ERROR;
  }
  uint64_t start = u->device_len; /* cached prefix served from the device tier */
  uint64_t nfresh = u->hist.n - p->reusable_len + p->delta;
  uint32_t* fresh = malloc((nfresh + 1) * sizeof(uint32_t));
  size_t k = 0;
  for (size_t i = p->reusable_len; i < u->hist.n; ++i) fresh[k++] = u->hist.v[i];
  for (uint32_t i = 0; i < p->delta; ++i) fresh[k++] = newtok[i];
  for (uint32_t i = 0; i < p->delta; ++i) u32_push(&u->hist, newtok[i]);
  double* ck = malloc((start * L * d + 1) * sizeof(double));
  double* cv = malloc((start * L * d + 1) * sizeof(double));
  for (size_t l = 0; l < L; ++l)
    for (uint64_t pos = 0; pos < start; ++pos) {
      const double* src = u->kv.v + (pos * L + l) * 2 * d;
      memcpy(ck + (l * start + pos) * d, src, d * sizeof(double));
      memcpy(cv + (l * start + pos) * d, src + d, d * sizeof(double));
    }
  size_t M = nfresh + p->num_candidates;
  double* nk = malloc(L * M * d * sizeof(double));
  double* nv = malloc(L * M * d * sizeof(double));
  int rc = orc_forward(&e->model, ck, cv, start, fresh, (uint32_t)nfresh, cands,
                       p->num_candidates, logits, nk, nv);
  if (rc == ORC_OK) {
    uint64_t newlen = start + nfresh;
    f64_reserve(&u->kv, newlen * L * 2 * d);
    for (uint64_t i = 0; i < nfresh; ++i)
      for (size_t l = 0; l < L; ++l) {
        double* dst = u->kv.v + ((start + i) * L + l) * 2 * d;
        memcpy(dst, nk + (l * M + i) * d, d * sizeof(double));
        memcpy(dst + d, nv + (l * M + i) * d, d * sizeof(double));
      }
    if (newlen > u->kv_len) u->kv_len = newlen;
  } else {
    snprintf(e->err, sizeof e->err, "forward: bad token or no candidates");
  }
  free(fresh); free(ck); free(cv); free(nk); free(nv);
  return rc;
}

/* Value backend, recompute mode: full forward over the whole history. */
static int encode_recompute(orc_engine* e, int s, const uint32_t* newtok, uint32_t dn,
                            const uint32_t* cands, uint32_t nc, double* logits) {
  user_t* u = &e->users[s];
  for (uint32_t i = 0; i < dn; ++i) u32_push(&u->hist, newtok[i]);
  int rc = orc_forward(&e->model, NULL, NULL, 0, u->hist.v, (uint32_t)u->hist.n, cands, nc,
                       logits, NULL, NULL);
  if (rc != ORC_OK) snprintf(e->err, sizeof e->err, "forward: bad token or no candidates");
  return rc;
}

int orc_process_batch(orc_engine* e, uint32_t n, const uint64_t* ts, const uint32_t* users,
                      const uint32_t* dn, const uint32_t* nc, const uint32_t* tokens,
                      const uint32_t* cands) {
  (void)ts;
  e->n_plans = 0;
  e->n_evs = 0;
  e->n_logit_rows = 0;
  e->n_scratch = 0; /* a rejected batch leaks its scratch pages, as the reference does */
  e->err[0] = 0;
  if (n == 0) return ORC_OK;
  const int hier = e->mode == ORC_HIERARCHICAL;
  const int cached = e->mode != ORC_RECOMPUTE;
  const uint32_t L = e->kv.num_layers;
  const double start = e->clock;
  int rc = complete_due(e, start);
  if (rc) return rc;
  double t = start, st[9] = {0};

  if (e->cap_plans < n) {
    e->cap_plans = n;
    e->plans = realloc(e->plans, n * sizeof(orc_plan));
  }
  /* ---- metadata (manager.cpp:74 prepare_metadata) ---- */
  int* slot = malloc(n * sizeof(int));
  if (cached) {
    for (uint32_t i = 0; i < n; ++i) slot[i] = get_slot(e, users[i]);
    unsigned char* inb = calloc(e->n_users + 1, 1);
    uint64_t* proj_total = malloc(n * sizeof(uint64_t));
    uint64_t* proj_dev = malloc(n * sizeof(uint64_t));
    int* first = malloc(n * sizeof(int));
    for (uint32_t i = 0; i < n; ++i) inb[slot[i]] = 1;
    uint64_t need_total = 0;
    for (uint32_t i = 0; i < n; ++i) {
      user_t* u = &e->users[slot[i]];
      u->known = 1;
      u->last_access = ++e->clockc;
      lru_touch(e, slot[i]);
      first[i] = (int)i;
      for (uint32_t j = 0; j < i; ++j)
        if (slot[j] == slot[i]) { first[i] = first[j]; break; }
      if (first[i] == (int)i) {
        proj_total[i] = u->total_len;
        proj_dev[i] = u->device_len;
      }
      uint64_t prior = proj_total[first[i]], devlen = proj_dev[first[i]];
      orc_plan* p = &e->plans[e->n_plans++];
      memset(p, 0, sizeof(*p));
      p->user = users[i];
      p->history_len = prior;
      p->delta = dn[i];
      p->num_candidates = nc[i];
      if (nc[i] < 1) {
        snprintf(e->err, sizeof e->err, "request: need at least one candidate");
        free(inb); free(proj_total); free(proj_dev); free(first); free(slot);
        return ORC_ERROR;
      }
      if (devlen > 0) {
        p->device_served = devlen < prior ? devlen : prior;
        p->reusable_len = p->device_served;
      } else if (hier && u->persisted_len > 0) {
        p->host_onload = u->persisted_len;
        p->reusable_len = u->persisted_len;
        p->onload_chunks = (uint32_t)(u->persisted_len / e->kv.chunk_size);
      }
      p->fresh_history = prior - p->reusable_len;
      uint64_t target = prior + p->delta;
      uint64_t want = ceil_div(target, e->kv.page_size);
      uint64_t have = u->has_pages ? u->pages.n : 0;
      uint64_t grow = want > have ? want - have : 0;
      uint64_t scratch = ceil_div(p->num_candidates, e->kv.page_size);
      need_total += grow + scratch;
      if (need_total > e->kv.device_pages) {
        snprintf(e->err, sizeof e->err, "batch exceeds total device pages");
        free(inb); free(proj_total); free(proj_dev); free(first); free(slot);
        return ORC_REJECTED;
      }
      rc = make_room(e, grow + scratch, inb);
      if (rc) {
        free(inb); free(proj_total); free(proj_dev); free(first); free(slot);
        return rc;
      }
      u = &e->users[slot[i]];
      u->has_pages = 1;
      for (uint64_t g = 0; g < grow; ++g) u32_push(&u->pages, page_pop(e));
      for (uint64_t g = 0; g < scratch; ++g) {
        if (e->n_scratch == e->cap_scratch) {
          e->cap_scratch = e->cap_scratch ? 2 * e->cap_scratch : 64;
          e->scratch = realloc(e->scratch, e->cap_scratch * sizeof(uint32_t));
        }
        e->scratch[e->n_scratch++] = page_pop(e);
      }
      p->scratch_pages = (uint32_t)scratch;
      proj_total[first[i]] = target;
      proj_dev[first[i]] = p->reusable_len + p->fresh_history + p->delta;
    }
    free(inb); free(proj_total); free(proj_dev); free(first);
    st[0] = e->cost.meta_fixed;
  } else {
    for (uint32_t i = 0; i < n; ++i) {
      slot[i] = get_slot(e, users[i]);
      user_t* u = &e->users[slot[i]];
      orc_plan* p = &e->plans[e->n_plans++];
      memset(p, 0, sizeof(*p));
      p->user = users[i];
      p->history_len = u->recompute_len;
      p->delta = dn[i];
      p->num_candidates = nc[i];
      p->fresh_history = p->history_len;
      u->recompute_len += dn[i];
    }
  }
  if (e->occupied > e->peak_pages) e->peak_pages = e->occupied;
  t += st[0];

  /* ---- onload (sim.hpp:361-383): schedule + staging-capacity check ---- */
  size_t total_chunks = 0;
  for (size_t i = 0; i < e->n_plans; ++i) total_chunks += e->plans[i].onload_chunks;
  double* fire = malloc((L ? L : 1) * sizeof(double));
  schedule_onload(e, t, total_chunks, fire);
  if ((uint64_t)total_chunks * e->kv.chunk_size > (uint64_t)e->kv.onload_pages * e->kv.page_size) {
    snprintf(e->err, sizeof e->err, "onload buffer: batch exceeds staging capacity");
    free(fire); free(slot);
    return ORC_ERROR;
  }

  uint64_t fresh_total = 0;
  for (size_t i = 0; i < e->n_plans; ++i) {
    const orc_plan* p = &e->plans[i];
    fresh_total += p->fresh_history + p->delta + p->num_candidates;
  }
  if (cached) st[1] = e->cost.strip_fixed;
  st[2] = e->cost.embed_fixed + e->cost.embed_coeff * (double)fresh_total;
  st[3] = e->cost.layout_fixed + e->cost.layout_coeff * (double)fresh_total;
  if (cached) {
    st[4] = e->cost.await_fixed;
    st[5] = e->cost.update_fixed + e->cost.commit_per_chunk * (double)total_chunks;
  }
  t += st[1] + st[2] + st[3] + st[4] + st[5];

  if (cached)
    for (size_t i = 0; i < e->n_plans; ++i)
      if (e->plans[i].onload_chunks > 0) e->users[slot[i]].device_len = e->plans[i].reusable_len;

  /* ---- step 8 time charge ---- */
  double dom = 0;
  for (size_t i = 0; i < e->n_plans; ++i) {
    const orc_plan* p = &e->plans[i];
    double fresh = (double)(p->fresh_history + p->delta + p->num_candidates);
    double total = (double)(p->history_len + p->delta + p->num_candidates);
    double a = e->cost.attn_coeff * fresh * total;
    double lin = e->cost.linear_coeff * fresh;
    if (a + lin > dom) dom = a + lin;
  }
  double layer_comp = (double)n * dom;
  for (uint32_t l = 0; l < L; ++l) {
    double w = fire[l] - t;
    if (w < 0.0) w = 0.0;
    t += w;
    e->wait_sum += w;
    t += layer_comp;
    e->comp_sum += layer_comp;
    st[6] += w + layer_comp;
  }
  free(fire);

  /* ---- encode + append ---- */
  if (e->value) {
    const size_t V = e->model.vocab;
    free(e->logits);
    e->logits = malloc((size_t)n * V * sizeof(double));
  }
  size_t tok_off = 0, cand_off = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const orc_plan* p = &e->plans[i];
    if (cached) {
      user_t* u = &e->users[slot[i]];
      if (e->value) {
        rc = encode_value(e, slot[i], p, tokens + tok_off, cands + cand_off,
                          e->logits + (size_t)i * e->model.vocab);
        if (rc) { free(slot); return rc; }
        e->n_logit_rows++;
      }
      u = &e->users[slot[i]];
      u->device_len += p->fresh_history + p->delta;
      if (u->device_len > u->total_len) u->total_len = u->device_len;
    } else if (e->value) {
      rc = encode_recompute(e, slot[i], tokens + tok_off, dn[i], cands + cand_off, nc[i],
                            e->logits + (size_t)i * e->model.vocab);
      if (rc) { free(slot); return rc; }
      e->n_logit_rows++;
    }
    tok_off += dn[i];
    cand_off += nc[i];
  }
  /* ---- candidate scratch pages back to the stack (manager.cpp:196) ---- */
  if (cached)
    for (size_t i = 0; i < e->n_scratch; ++i) page_push(e, e->scratch[i]);
  e->n_scratch = 0;

  /* ---- step 9: proactive offload (sim.hpp:433) ---- */
  if (hier) {
    st[7] = e->cost.offload_submit;
    for (uint32_t i = 0; i < n; ++i) offload_ready_chunks(e, slot[i], t);
    t += st[7];
  }
  st[8] = e->cost.post_fixed;
  t += st[8];

  e->clock = t;
  e->latency_sum += t - start;
  for (int i = 0; i < 9; ++i) e->step_sum[i] += st[i];
  e->batches++;
  e->requests += n;
  for (size_t i = 0; i < e->n_plans; ++i) {
    const orc_plan* p = &e->plans[i];
    if (p->history_len > 0) {
      e->required += p->history_len;
      e->dev_served += p->device_served;
      e->host_served += p->host_onload;
    }
    e->tokens_processed += p->fresh_history + p->delta + p->num_candidates;
  }
  free(slot);
  return ORC_OK;
}

void orc_drain(orc_engine* e) { complete_due(e, 1e300); }

uint32_t orc_last_plans(const orc_engine* e, orc_plan* out, uint32_t cap) {
  uint32_t n = (uint32_t)e->n_plans;
  if (out) memcpy(out, e->plans, (n < cap ? n : cap) * sizeof(orc_plan));
  return n;
}

uint32_t orc_last_evictions(const orc_engine* e, orc_eviction* out, uint32_t cap) {
  uint32_t n = (uint32_t)e->n_evs;
  if (out) memcpy(out, e->evs, (n < cap ? n : cap) * sizeof(orc_eviction));
  return n;
}

uint32_t orc_last_logits(const orc_engine* e, double* out, uint32_t cap_rows) {
  uint32_t n = (uint32_t)e->n_logit_rows;
  if (out && e->logits)
    memcpy(out, e->logits, (size_t)(n < cap_rows ? n : cap_rows) * e->model.vocab * sizeof(double));
  return n;
}

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

uint32_t orc_known_users(const orc_engine* e, uint32_t* out, uint32_t cap) {
  uint32_t n = 0;
  for (size_t s = 0; s < e->n_users; ++s)
    if (e->users[s].known) {
      if (out && n < cap) out[n] = e->users[s].id;
      n++;
    }
  if (out) qsort(out, n < cap ? n : cap, sizeof(uint32_t), cmp_u32);
  return n;
}

int orc_user_state_get(const orc_engine* e, uint32_t user, orc_user_state* out) {
  int s = find_slot(e, user);
  if (s < 0 || !e->users[s].known) return ORC_ERROR;
  const user_t* u = &e->users[s];
  out->total_len = u->total_len;
  out->device_len = u->device_len;
  out->persisted_len = u->persisted_len;
  out->last_access = u->last_access;
  out->locked = (uint32_t)u->locked;
  out->num_pages = u->has_pages ? (uint32_t)u->pages.n : 0;
  out->host_chunks = u->host_chunks;
  out->pending_offload = u->pending;
  return ORC_OK;
}

uint32_t orc_user_pages(const orc_engine* e, uint32_t user, uint32_t* out, uint32_t cap) {
  int s = find_slot(e, user);
  if (s < 0 || !e->users[s].has_pages) return 0;
  const u32vec* p = &e->users[s].pages;
  if (out) memcpy(out, p->v, (p->n < cap ? p->n : cap) * sizeof(uint32_t));
  return (uint32_t)p->n;
}

uint32_t orc_lru_snapshot(const orc_engine* e, uint32_t* out, uint32_t cap) {
  uint32_t n = 0;
  for (int s = e->lru_head; s >= 0; s = e->users[s].next) {
    if (out && n < cap) out[n] = e->users[s].id;
    n++;
  }
  return n;
}

void orc_report_get(const orc_engine* e, orc_report* r) {
  memset(r, 0, sizeof(*r));
  const double nb = e->batches ? (double)e->batches : 1.0;
  for (int i = 0; i < 9; ++i) r->step_ms[i] = e->step_sum[i] / nb * 1e3;
  r->wait_ms = e->wait_sum / nb * 1e3;
  r->comp_ms = e->comp_sum / nb * 1e3;
  if (e->required == 0) {
    r->gpu_hit_ratio = 1.0;
    r->total_hit_ratio = 1.0;
  } else {
    r->gpu_hit_ratio = (double)e->dev_served / (double)e->required;
    r->total_hit_ratio = (double)(e->dev_served + e->host_served) / (double)e->required;
  }
  r->tokens_processed = e->tokens_processed;
  r->evictions = e->evictions;
  r->tail_tokens_lost = e->tail_lost;
  r->requests = e->requests;
  r->batches = e->batches;
  r->avg_latency_ms = e->latency_sum / nb * 1e3;
  r->total_latency_ms = e->latency_sum * 1e3;
  r->peak_pages = e->peak_pages;
  r->pages_allocated = e->pages_allocated;
  r->occupied_pages = e->occupied;
  r->free_pages = e->stack_n;
  r->quota_in_flight = e->quota_in_flight;
  r->clock = e->clock;
}

int orc_evict_user(orc_engine* e, uint32_t user) {
  int s = find_slot(e, user);
  if (s < 0) { snprintf(e->err, sizeof e->err, "evict: unknown user"); return ORC_ERROR; }
  return evict(e, s, NULL);
}

int orc_is_locked(const orc_engine* e, uint32_t user) {
  int s = find_slot(e, user);
  return s >= 0 && e->users[s].locked;
}
