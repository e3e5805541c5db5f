// extern "C" boundary (include/mtkv_b200.h). Thin: validates, forwards to the
// planner / engine, converts failures into return codes + mtkv_last_error().
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "engine.hpp"
#include "planner.hpp"

#include "workload.hpp"

using namespace mtkv_b200;

static thread_local std::string g_err;

namespace mtkv_b200 {
void set_last_error(const std::string& m) { g_err = m; }
}  // namespace mtkv_b200

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

struct mtkv_planner {
  Planner p;
  mtkv_planner(const mtkv_kv_config& kv, const mtkv_cost_model& c, int mode) : p(kv, c, mode, false) {}
};
struct mtkv_engine {
  Engine e;
  mtkv_engine(const mtkv_kv_config& kv, const mtkv_cost_model& c, const mtkv_engine_options& o) : e(kv, c, o) {}
};

static const Planner* planner_of(const void* obj, int is_engine) {
  if (!obj) return nullptr;
  return is_engine ? &static_cast<const mtkv_engine*>(obj)->e.planner : &static_cast<const mtkv_planner*>(obj)->p;
}
static Planner* planner_of(void* obj, int is_engine) {
  if (!obj) return nullptr;
  return is_engine ? &static_cast<mtkv_engine*>(obj)->e.planner : &static_cast<mtkv_planner*>(obj)->p;
}

static std::string validate(const mtkv_kv_config& c) {
  if (c.page_size < 1) return "config: page_size must be >= 1";
  if (c.chunk_size < c.page_size) return "config: chunk_size must be >= page_size";
  if (c.chunk_size % c.page_size) return "config: chunk_size must be a multiple of page_size";
  if (c.device_pages < 1) return "config: device_pages must be >= 1";
  if (c.offload_quota < c.chunk_size) return "config: offload_quota must admit at least one chunk";
  if (c.num_layers < 1 || c.num_heads < 1 || c.head_dim < 1) return "config: model dimensions must be positive";
  if (c.bytes_per_element < 1) return "config: bytes_per_element must be >= 1";
  return "";
}

static std::string validate_cost(const mtkv_cost_model& c) {
  if (!(c.bus_bandwidth > 0 && c.host_bandwidth > 0)) return "cost model: bandwidths must be positive";
  if (!(c.tx_setup >= 0 && c.page_op >= 0 && c.attn_coeff >= 0 && c.linear_coeff >= 0 && c.embed_coeff >= 0 &&
        c.layout_coeff >= 0))
    return "cost model: coefficients must be nonnegative";
  return "";
}

extern "C" {

const char* mtkv_last_error(void) { return g_err.c_str(); }

void mtkv_kv_config_default(mtkv_kv_config* o) {
  *o = mtkv_kv_config{8, 4, 128, 32, 1024, 40960, 10008, 2, 8192, 0};
}

int mtkv_kv_config_validate(const mtkv_kv_config* c) {
  std::string e = validate(*c);
  return e.empty() ? MTKV_OK : fail(MTKV_ERROR, e);
}

void mtkv_cost_model_default(mtkv_cost_model* o) {
  *o = mtkv_cost_model{25e9, 10e-6, 50e9, 50e-9, 2e-10, 1e-7, 5e-8, 5e-8, 1e-4, 5e-5,
                       1e-4, 1e-4, 5e-5, 5e-5, 5e-6, 3e-5, 2e-4};
}

uint64_t mtkv_pages_needed(uint64_t len, uint32_t page_size) {
  if (page_size < 1) { g_err = "pages_needed: page size must be >= 1"; return 0; }
  return (len + page_size - 1) / page_size;
}

uint64_t mtkv_persisted_prefix(uint64_t len, uint32_t chunk_size) {
  if (chunk_size < 1) { g_err = "persisted_prefix: chunk size must be >= 1"; return 0; }
  return (len / chunk_size) * chunk_size;
}

static std::string trim(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r\n");
  if (b == std::string::npos) return "";
  return s.substr(b, s.find_last_not_of(" \t\r\n") - b + 1);
}

int mtkv_parse_config_text(const char* text, const char* origin, mtkv_kv_config* out) {
  mtkv_kv_config c;
  mtkv_kv_config_default(&c);
  std::istringstream in(text ? text : "");
  std::string line, org = origin ? origin : "config";
  int ln = 0;
  while (std::getline(in, line)) {
    ++ln;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    line = trim(line);
    if (line.empty()) continue;
    const auto eq = line.find('=');
    const std::string where = org + ":" + std::to_string(ln);
    if (eq == std::string::npos) return fail(MTKV_ERROR, where + ": expected key=value");
    const std::string key = trim(line.substr(0, eq)), val = trim(line.substr(eq + 1));
    uint64_t n = 0;
    try {
      n = std::stoull(val);
    } catch (...) {
      return fail(MTKV_ERROR, where + ": bad number '" + val + "'");
    }
    if (key == "num_layers") c.num_layers = uint32_t(n);
    else if (key == "num_heads") c.num_heads = uint32_t(n);
    else if (key == "head_dim") c.head_dim = uint32_t(n);
    else if (key == "page_size") c.page_size = uint32_t(n);
    else if (key == "chunk_size") c.chunk_size = uint32_t(n);
    else if (key == "device_pages") c.device_pages = uint32_t(n);
    else if (key == "onload_pages") c.onload_pages = uint32_t(n);
    else if (key == "bytes_per_element") c.bytes_per_element = uint32_t(n);
    else if (key == "offload_quota") c.offload_quota = n;
    else if (key == "host_capacity") c.host_capacity = n;
    else return fail(MTKV_ERROR, where + ": unknown key '" + key + "'");
  }
  std::string e = validate(c);
  if (!e.empty()) return fail(MTKV_ERROR, e);
  *out = c;
  return MTKV_OK;
}

// ---------------------------------------------------------------- planner --
mtkv_planner* mtkv_planner_create(const mtkv_kv_config* kv, const mtkv_cost_model* cost, int mode) {
  std::string e = validate(*kv);
  if (e.empty()) e = validate_cost(*cost);
  if (!e.empty()) { g_err = e; return nullptr; }
  if (mode < 0 || mode > 2) { g_err = "unknown mode"; return nullptr; }
  return new mtkv_planner(*kv, *cost, mode);
}

void mtkv_planner_destroy(mtkv_planner* p) { delete p; }

int mtkv_planner_process_batch(mtkv_planner* p, const mtkv_request* reqs, uint32_t n) {
  BatchWork w;
  p->p.plan_batch(reqs, n, w);
  p->p.keep_last(w);
  return w.rc ? fail(w.rc, w.error) : MTKV_OK;
}

int mtkv_planner_drain(mtkv_planner* p) {
  p->p.drain();
  return MTKV_OK;
}

int mtkv_planner_set_onload_policy(mtkv_planner* p, uint32_t policy, double onload_gbs, double recompute_mtok_s) {
  if (!p) return fail(MTKV_ERROR, "planner: null handle");
  if (policy > MTKV_ONLOAD_ADAPTIVE || onload_gbs <= 0 || recompute_mtok_s <= 0)
    return fail(MTKV_ERROR, "planner: onload policy needs a known policy and positive rates");
  p->p.set_onload_policy(int(policy), onload_gbs * 1e9, recompute_mtok_s * 1e6);
  return MTKV_OK;
}

int mtkv_planner_prepare_metadata(mtkv_planner* p, const mtkv_request* reqs, uint32_t n, int host_enabled) {
  std::string err;
  const int rc = p->p.mgr_prepare(reqs, n, host_enabled != 0, err);
  return rc ? fail(rc, err) : MTKV_OK;
}

uint32_t mtkv_planner_scratch_pages(const mtkv_planner* p, uint32_t req, uint32_t* out, uint32_t cap) {
  const std::vector<uint32_t>* v = p->p.mgr_scratch(req);
  if (!v) return 0;
  for (uint32_t i = 0; out && i < v->size() && i < cap; ++i) out[i] = (*v)[i];
  return uint32_t(v->size());
}

#define MTKV_STEP(call)            \
  do {                             \
    std::string err;               \
    const int rc = (call);         \
    return rc ? fail(rc, err) : MTKV_OK; \
  } while (0)

int mtkv_planner_release_scratch(mtkv_planner* p, const uint32_t* pages, uint32_t n) {
  MTKV_STEP(p->p.mgr_release_pages(pages, n, err));
}
int mtkv_planner_commit_onload(mtkv_planner* p, uint32_t user, uint64_t reusable_len, uint32_t onload_chunks) {
  MTKV_STEP(p->p.mgr_commit_onload(user, reusable_len, onload_chunks, err));
}
int mtkv_planner_finish_append(mtkv_planner* p, uint32_t user, uint64_t appended) {
  MTKV_STEP(p->p.mgr_finish_append(user, appended, err));
}
int mtkv_planner_advance_persisted(mtkv_planner* p, uint32_t user, uint64_t tokens) {
  MTKV_STEP(p->p.mgr_advance_persisted(user, tokens, err));
}
int mtkv_planner_lock_user(mtkv_planner* p, uint32_t user) { MTKV_STEP(p->p.mgr_lock(user, true, err)); }
int mtkv_planner_unlock_user(mtkv_planner* p, uint32_t user) { MTKV_STEP(p->p.mgr_lock(user, false, err)); }
uint32_t mtkv_planner_last_page_len(const mtkv_planner* p, uint32_t user) { return p->p.last_page_len(user); }

// ----------------------------------------------------------------- engine --
mtkv_engine* mtkv_engine_create(const mtkv_kv_config* kv, const mtkv_cost_model* cost,
                                const mtkv_engine_options* opts) {
  std::string e = validate(*kv);
  if (e.empty()) e = validate_cost(*cost);
  if (!e.empty()) { g_err = e; return nullptr; }
  if (opts->backend == MTKV_BACKEND_VALUE) {
    const auto& m = opts->model;
    if (m.num_layers != kv->num_layers || m.num_heads * m.head_dim != kv->num_heads * kv->head_dim) {
      g_err = "value backend: model dimensions disagree with cache config";
      return nullptr;
    }
    if (m.vocab < 1) { g_err = "value backend: vocab must be >= 1"; return nullptr; }
  }
  auto* eng = new mtkv_engine(*kv, *cost, *opts);
  std::string err;
  if (int rc = eng->e.init(err)) {
    (void)rc;
    delete eng;
    g_err = err;
    return nullptr;
  }
  return eng;
}

void mtkv_engine_destroy(mtkv_engine* e) { delete e; }

int mtkv_engine_process_batch(mtkv_engine* e, const mtkv_request* reqs, uint32_t n) {
  std::string err;
  const int rc = e->e.process_batch(reqs, n, err);
  return rc ? fail(rc, err) : MTKV_OK;
}

int mtkv_engine_run(mtkv_engine* e, const mtkv_request* trace, uint64_t n, mtkv_run_report* out) {
  // sim.hpp:135 run(): batchify (workload.cpp:247), every batch, drain, report
  const uint64_t bs = e->e.batch_size();
  std::string err;
  for (uint64_t i = 0; i < n; i += bs) {
    const uint32_t m = uint32_t(n - i < bs ? n - i : bs);
    const int rc = e->e.process_batch(trace + i, m, err);
    if (rc) return fail(rc, err);
  }
  e->e.drain(err);
  if (out) e->e.report(*out);
  return MTKV_OK;
}

int mtkv_engine_drain(mtkv_engine* e) {
  std::string err;
  const int rc = e->e.drain(err);
  return rc ? fail(rc, err) : MTKV_OK;
}

int mtkv_engine_synchronize(mtkv_engine* e) {
  std::string err;
  const int rc = e->e.synchronize(err);
  return rc ? fail(rc, err) : MTKV_OK;
}

int mtkv_engine_last_logits(mtkv_engine* e, float* out, uint32_t cap_rows) {
  std::string err;
  const int rc = e->e.last_logits(out, cap_rows, err);
  if (!err.empty()) {
    g_err = err;
    return -1;
  }
  return rc;
}

int mtkv_engine_last_rankings(mtkv_engine* e, uint32_t* out, uint64_t cap) {
  std::string err;
  const int rc = e->e.last_rankings(out, cap, err);
  return !err.empty() ? (fail(MTKV_ERROR, err), -1) : rc;
}

int mtkv_engine_batch_rankings(mtkv_engine* e, uint64_t ticket, uint32_t* out, uint64_t cap) {
  std::string err;
  const int rc = e->e.batch_rankings(ticket, out, cap, err);
  return !err.empty() ? (fail(MTKV_ERROR, err), -1) : rc;
}

uint64_t mtkv_engine_batches_submitted(const mtkv_engine* e) { return e->e.batches_submitted(); }

void mtkv_engine_last_plan_ms(const mtkv_engine* e, double* plan_ms, double* ctl_kernel_ms) {
  e->e.last_plan_ms(plan_ms, ctl_kernel_ms);
}

int mtkv_engine_check_conservation(mtkv_engine* e) {
  std::string err;
  const int rc = e->e.check_conservation(err);
  return rc ? fail(rc, err) : MTKV_OK;
}

int64_t mtkv_engine_read_user_kv(mtkv_engine* e, uint32_t user, uint32_t layer, uint16_t* k, uint16_t* v,
                                 uint64_t cap) {
  std::string err;
  const int64_t n = e->e.read_user_kv(user, layer, k, v, cap, err);
  if (n < 0) g_err = err;
  return n;
}

double mtkv_engine_last_batch_ms(mtkv_engine* e) { return e->e.last_batch_ms(); }
double mtkv_engine_last_attention_ms(mtkv_engine* e, uint32_t* launches) { return e->e.last_attention_ms(launches); }
double mtkv_engine_last_proj_ms(mtkv_engine* e, uint32_t* launches, uint64_t* rows) {
  return e->e.last_proj_ms(launches, rows);
}
int mtkv_engine_last_chunk_copy_ms(mtkv_engine* e, double* scatter_ms, uint32_t* scatter_chunks, double* gather_ms,
                                   uint32_t* gather_chunks) {
  return e->e.last_chunk_copy_ms(scatter_ms, scatter_chunks, gather_ms, gather_chunks);
}
uint64_t mtkv_engine_kernel_launches(const mtkv_engine* e) { return e->e.launches; }
void mtkv_engine_set_profile(mtkv_engine* e, uint32_t on) { e->e.set_profile(on); }
int mtkv_engine_set_onload_policy(mtkv_engine* e, uint32_t policy, double onload_gbs, double recompute_mtok_s) {
  std::string err;
  const int rc = e->e.set_onload_policy(policy, onload_gbs, recompute_mtok_s, err);
  return rc ? fail(rc, err) : MTKV_OK;
}

// ------------------------------------------------------------ manager view --
int mtkv_report(const void* obj, int is_engine, mtkv_run_report* out) {
  if (!obj) return fail(MTKV_ERROR, "null object");
  if (is_engine) static_cast<const mtkv_engine*>(obj)->e.report(*out);
  else planner_of(obj, 0)->report(*out);
  return MTKV_OK;
}

uint32_t mtkv_last_plans(const void* obj, int is_engine, mtkv_request_plan* out, uint32_t cap) {
  const auto& w = planner_of(obj, is_engine)->last();
  const uint32_t n = uint32_t(w.reqs.size());
  for (uint32_t i = 0; out && i < n && i < cap; ++i) out[i] = w.reqs[i].plan;
  return n;
}

uint32_t mtkv_last_evictions(const void* obj, int is_engine, mtkv_eviction* out, uint32_t cap) {
  const auto& w = planner_of(obj, is_engine)->last();
  const uint32_t n = uint32_t(w.evictions.size());
  for (uint32_t i = 0; out && i < n && i < cap; ++i) out[i] = w.evictions[i];
  return n;
}

uint32_t mtkv_known_users(const void* obj, int is_engine, uint32_t* out, uint32_t cap) {
  auto v = planner_of(obj, is_engine)->known_users();
  for (uint32_t i = 0; out && i < v.size() && i < cap; ++i) out[i] = v[i];
  return uint32_t(v.size());
}

int mtkv_user_state(const void* obj, int is_engine, uint32_t user, mtkv_sequence_state* out) {
  const UserRec* u = planner_of(obj, is_engine)->find(user);
  if (!u || !u->known) return fail(MTKV_ERROR, "unknown user");
  out->total_len = u->total_len;
  out->device_len = u->device_len;
  out->persisted_len = u->persisted_len;
  out->last_access = u->last_access;
  out->locked = u->locked;
  out->num_pages = u->has_pages ? uint32_t(u->pages.size()) : 0;
  out->host_chunks = uint32_t(u->host_chunks.size());
  out->pending_offload = u->pending;
  return MTKV_OK;
}

uint32_t mtkv_user_pages(const void* obj, int is_engine, uint32_t user, uint32_t* out, uint32_t cap) {
  const UserRec* u = planner_of(obj, is_engine)->find(user);
  if (!u || !u->has_pages) return 0;
  for (uint32_t i = 0; out && i < u->pages.size() && i < cap; ++i) out[i] = u->pages[i];
  return uint32_t(u->pages.size());
}

uint32_t mtkv_lru_snapshot(const void* obj, int is_engine, uint32_t* out, uint32_t cap) {
  auto v = planner_of(obj, is_engine)->lru_snapshot();
  for (uint32_t i = 0; out && i < v.size() && i < cap; ++i) out[i] = v[i];
  return uint32_t(v.size());
}

int mtkv_evict_user(void* obj, int is_engine, uint32_t user) {
  std::string err;
  const int rc = planner_of(obj, is_engine)->evict(user, err);
  return rc ? fail(rc, err) : MTKV_OK;
}

int mtkv_is_locked(const void* obj, int is_engine, uint32_t user) {
  const UserRec* u = planner_of(obj, is_engine)->find(user);
  return u && u->locked ? 1 : 0;
}

uint64_t mtkv_get_total_cache_length(const void* obj, int is_engine, uint32_t user) {
  const UserRec* u = planner_of(obj, is_engine)->find(user);
  if (!u || !u->known) return 0;
  return u->device_len > u->persisted_len ? u->device_len : u->persisted_len;
}

char* mtkv_dump_page_map(const void* obj, int is_engine) {
  const Planner* p = planner_of(obj, is_engine);
  std::string s = "{";
  bool first = true;
  for (uint32_t u : p->known_users()) {
    if (!first) s += ",";
    first = false;
    s += "\"" + std::to_string(u) + "\":[";
    const UserRec* r = p->find(u);
    if (r && r->has_pages)
      for (size_t i = 0; i < r->pages.size(); ++i) {
        if (i) s += ",";
        s += std::to_string(r->pages[i]);
      }
    s += "]";
  }
  s += "}";
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

int64_t mtkv_state_blob(const void* obj, int is_engine, uint8_t* buf, uint64_t cap) {
  const Planner* p = planner_of(obj, is_engine);
  std::vector<uint8_t> b;
  b.reserve(1 << 16);
  auto put = [&b](const void* x, size_t n) {
    const uint8_t* c = static_cast<const uint8_t*>(x);
    b.insert(b.end(), c, c + n);
  };
  auto u32 = [&put](uint32_t x) { put(&x, 4); };
  auto u64 = [&put](uint64_t x) { put(&x, 8); };
  put("MTKVST01", 8);
  const std::vector<uint32_t> users = p->known_users();
  u64(users.size());
  for (uint32_t id : users) {
    const UserRec* u = p->find(id);
    u32(id);
    u32(u->locked ? 1 : 0);
    u64(u->total_len);
    u64(u->device_len);
    u64(u->persisted_len);
    u64(u->last_access);
    u64(u->host_chunks.size());
    u64(u->pending);
    const size_t np = u->has_pages ? u->pages.size() : 0;
    u64(np);
    if (np) put(u->pages.data(), np * 4);
  }
  const std::vector<uint32_t> lru = p->lru_snapshot();
  u64(lru.size());
  if (!lru.empty()) put(lru.data(), lru.size() * 4);
  mtkv_run_report r;
  if (is_engine) static_cast<const mtkv_engine*>(obj)->e.report(r);
  else p->report(r);
  u64(r.evictions);
  u64(r.tail_tokens_lost);
  u64(r.pages_allocated);
  u64(r.occupied_pages);
  u64(r.free_pages);
  u64(r.quota_in_flight);
  put(&r.clock, 8);
  if (buf) std::memcpy(buf, b.data(), std::min<uint64_t>(cap, b.size()));
  return int64_t(b.size());
}

// --------------------------------------------------------------- workload --
void mtkv_gen_config_default(mtkv_gen_config* g) {
  *g = mtkv_gen_config{100, 2000, 0, 9.0, 1.5, 1.3, 1000.0, 6375.0, 1, 20000, 0, 5, 0, 42};
}

int mtkv_gen_config_preset(const char* name, mtkv_gen_config* g) {
  mtkv_gen_config_default(g);
  const std::string n = name ? name : "";
  if (n == "kuairand1k") {
    g->num_users = 1000; g->total_requests = 20000; g->mean_final_len = 6375; g->min_len = 1; g->max_len = 20000;
  } else if (n == "mt") {
    g->num_users = 2884; g->total_requests = 20000; g->mean_final_len = 5189; g->min_len = 4000; g->max_len = 6000;
  } else {
    return fail(MTKV_ERROR, "unknown preset '" + n + "' (expected kuairand1k or mt)");
  }
  g->gap_log_mu = 9.0;
  g->gap_log_sigma = 1.6;
  g->candidates = 5;
  g->seed = 42;
  return MTKV_OK;
}

char* mtkv_generate_trace_jsonl(const mtkv_gen_config* g) {
  std::vector<TraceRec> tr;
  std::string err;
  if (generate(*g, tr, err)) { g_err = err; return nullptr; }
  const std::string s = to_jsonl(tr);
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

void mtkv_free(void* p) { std::free(p); }

}  // extern "C"
