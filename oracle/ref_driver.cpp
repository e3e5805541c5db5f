// Test infrastructure only (see oracle/README.md): a thin C-ABI driver over the
// UNMODIFIED reference library compiled from /root/reference/proj/core/src by
// oracle/Makefile into oracle/_ref/libmtkv_ref.so. It is never linked into the
// product; tests/, bench.py's cpu_baseline / --impl reference leg and the golden
// fixture generator (tools/make_golden.py) are its only callers.
//
// Entry point: mtkv_ref_call(json) -> json. Commands:
//   "gen_trace" : reference generate_trace()            (workload.cpp:85)
//   "run"       : reference Engine<B>::process_batch()   (sim.hpp:332) batch by
//                 batch, dumping the full manager state after every batch so the
//                 B200 engine's control plane can be compared bit-exactly.
//   "forward"   : reference forward_incremental()        (model.cpp:140)
//   "bench"     : bounded CPU baseline of the value-backend serving path,
//                 one reference Engine per host thread over a user shard.
#include <atomic>
#include <chrono>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include <json.hpp>

#include "mtkv/sim.hpp"

using nlohmann::json;
using namespace mtkv;

namespace {

KVConfig kv_from(const json& j) {
  KVConfig c;
  if (!j.is_object()) return c;
  if (j.contains("num_layers")) c.num_layers = j["num_layers"];
  if (j.contains("num_heads")) c.num_heads = j["num_heads"];
  if (j.contains("head_dim")) c.head_dim = j["head_dim"];
  if (j.contains("page_size")) c.page_size = j["page_size"];
  if (j.contains("chunk_size")) c.chunk_size = j["chunk_size"];
  if (j.contains("device_pages")) c.device_pages = j["device_pages"];
  if (j.contains("onload_pages")) c.onload_pages = j["onload_pages"];
  if (j.contains("bytes_per_element")) c.bytes_per_element = j["bytes_per_element"];
  if (j.contains("offload_quota")) c.offload_quota = j["offload_quota"];
  if (j.contains("host_capacity")) c.host_capacity = j["host_capacity"];
  return c;
}

CostModel cost_from(const json& j) {
  CostModel c;
  if (!j.is_object()) return c;
#define F(name) \
  if (j.contains(#name)) c.name = j[#name].get<double>();
  F(bus_bandwidth) F(tx_setup) F(host_bandwidth) F(page_op) F(attn_coeff)
  F(linear_coeff) F(embed_coeff) F(layout_coeff) F(meta_fixed) F(strip_fixed)
  F(embed_fixed) F(layout_fixed) F(await_fixed) F(update_fixed)
  F(commit_per_chunk) F(offload_submit) F(post_fixed)
#undef F
  return c;
}

ModelConfig model_from(const json& j) {
  ModelConfig m;
  if (!j.is_object()) return m;
  if (j.contains("num_layers")) m.num_layers = j["num_layers"];
  if (j.contains("num_heads")) m.num_heads = j["num_heads"];
  if (j.contains("head_dim")) m.head_dim = j["head_dim"];
  if (j.contains("vocab")) m.vocab = j["vocab"];
  if (j.contains("seed")) m.seed = j["seed"];
  return m;
}

std::vector<Request> trace_from(const json& j) {
  if (j.is_string()) return trace_from_jsonl(j.get<std::string>(), "json");
  std::vector<Request> out;
  for (const auto& r : j) {
    Request q;
    q.timestamp = r.value("ts", 0ull);
    q.user = r["user"];
    q.new_token_count = r["dn"];
    q.candidate_count = r["nc"];
    if (r.contains("tokens")) q.new_tokens = r["tokens"].get<std::vector<TokenId>>();
    if (r.contains("cands")) q.candidates = r["cands"].get<std::vector<TokenId>>();
    out.push_back(std::move(q));
  }
  return out;
}

GenConfig gen_from(const json& j) {
  GenConfig g;
  if (j.contains("preset")) g = resolve_preset(j["preset"]);
  if (j.contains("num_users")) g.num_users = j["num_users"];
  if (j.contains("total_requests")) g.total_requests = j["total_requests"];
  if (j.contains("mean_final_len")) g.mean_final_len = j["mean_final_len"];
  if (j.contains("min_len")) g.min_len = j["min_len"];
  if (j.contains("max_len")) g.max_len = j["max_len"];
  if (j.contains("fixed_delta")) g.fixed_delta = j["fixed_delta"];
  if (j.contains("candidates")) g.candidates = j["candidates"];
  if (j.contains("vocab")) g.vocab = j["vocab"];
  if (j.contains("seed")) g.seed = j["seed"];
  if (j.contains("gap_log_mu")) g.gap_log_mu = j["gap_log_mu"];
  if (j.contains("gap_log_sigma")) g.gap_log_sigma = j["gap_log_sigma"];
  if (j.contains("pareto")) g.family = j["pareto"].get<bool>() ? TailFamily::Pareto : TailFamily::LogNormal;
  return g;
}

Mode mode_from(const json& j) { return parse_mode(j.value("mode", std::string("hierarchical"))); }

// Complete control-plane state after a batch: every known user's lengths,
// lock bit, recency stamp, page list; counters; LRU order; free count.
template <class B>
json dump_state(Engine<B>& eng) {
  json users = json::array();
  auto& mgr = eng.manager();
  for (UserId u : mgr.known_users()) {
    const SequenceState* s = mgr.find(u);
    json ju;
    ju["user"] = u;
    ju["total_len"] = s->total_len;
    ju["device_len"] = s->device_len;
    ju["persisted_len"] = s->persisted_len;
    ju["locked"] = s->locked;
    ju["last_access"] = s->last_access;
    ju["pages"] = mgr.user_pages(u);
    ju["host_chunks"] = eng.host().chunk_count(u);
    ju["pending_offload"] = eng.pending_offload_chunks(u);
    users.push_back(std::move(ju));
  }
  json st;
  st["users"] = std::move(users);
  st["lru"] = mgr.lru().snapshot();
  st["evictions"] = mgr.counters().evictions;
  st["tail_tokens_lost"] = mgr.counters().tail_tokens_lost;
  st["pages_allocated"] = mgr.counters().pages_allocated;
  st["occupied_pages"] = mgr.occupied_pages();
  st["free_pages"] = eng.device().free_count();
  st["quota_in_flight"] = eng.quota().in_flight;
  st["clock"] = eng.clock();
  return st;
}

json report_json(const RunReport& r) { return json::parse(r.to_json()); }

// The canonical binary state image of include/mtkv_b200.h mtkv_state_blob,
// built here from the reference Engine's own accessors (independent encoder).
template <class B>
void state_blob(Engine<B>& eng, std::vector<std::uint8_t>& b) {
  b.clear();
  auto put = [&b](const void* x, std::size_t n) {
    const auto* c = static_cast<const std::uint8_t*>(x);
    b.insert(b.end(), c, c + n);
  };
  auto u32 = [&put](std::uint32_t x) { put(&x, 4); };
  auto u64 = [&put](std::uint64_t x) { put(&x, 8); };
  put("MTKVST01", 8);
  auto& mgr = eng.manager();
  const std::vector<UserId> users = mgr.known_users();
  u64(users.size());
  for (UserId u : users) {
    const SequenceState* s = mgr.find(u);
    u32(u);
    u32(s->locked ? 1 : 0);
    u64(s->total_len);
    u64(s->device_len);
    u64(s->persisted_len);
    u64(s->last_access);
    u64(eng.host().chunk_count(u));
    u64(eng.pending_offload_chunks(u));
    const auto& pages = mgr.user_pages(u);
    u64(pages.size());
    for (PageId pg : pages) u32(pg);
  }
  const auto lru = mgr.lru().snapshot();
  u64(lru.size());
  for (UserId u : lru) u32(u);
  u64(mgr.counters().evictions);
  u64(mgr.counters().tail_tokens_lost);
  u64(mgr.counters().pages_allocated);
  u64(mgr.occupied_pages());
  u64(eng.device().free_count());
  u64(eng.quota().in_flight);
  const double clk = eng.clock();
  put(&clk, 8);
}

using BlobCb = void (*)(std::uint64_t batch, const std::uint8_t* data, std::uint64_t n, int rejected);

// batch boundaries: explicit "batch_sizes" (a caller that batches a trace
// unevenly, e.g. bench.py's prefill vs revisit batches), else batchify
std::vector<std::vector<Request>> batches_of(const json& req, const std::vector<Request>& trace, std::uint32_t bs) {
  if (!req.contains("batch_sizes")) return batchify(trace, bs);
  std::vector<std::vector<Request>> out;
  std::size_t at = 0;
  for (std::size_t n : req["batch_sizes"].get<std::vector<std::size_t>>()) {
    if (at + n > trace.size()) throw Error("batch_sizes exceed the trace");
    out.emplace_back(trace.begin() + std::ptrdiff_t(at), trace.begin() + std::ptrdiff_t(at + n));
    at += n;
  }
  if (at != trace.size()) throw Error("batch_sizes do not cover the trace");
  return out;
}

template <class B>
json run_engine(const json& req, const std::vector<Request>& trace, BlobCb blob_cb = nullptr) {
  KVConfig kv = kv_from(req.value("kv", json::object()));
  CostModel cost = cost_from(req.value("cost", json::object()));
  EngineOptions opts;
  opts.mode = mode_from(req);
  opts.batch_size = req.value("batch_size", 1u);
  opts.seed = req.value("seed", 1ull);
  ModelParams params;
  std::vector<std::vector<double>> logits;
  std::vector<TraceEvent> events;
  if constexpr (std::is_same_v<B, ValueBackend>) {
    params = ModelParams::random(model_from(req.value("model", json::object())));
    opts.model = &params;
    opts.logit_sink = &logits;
  }
  const bool dump = !blob_cb && req.value("dump_state", true);
  std::vector<std::uint8_t> blob;
  std::uint64_t bi = 0;
  const bool want_events = req.value("events", false);
  if (want_events) opts.event_sink = &events;
  Engine<B> eng(kv, cost, opts);
  json out;
  json batches = json::array();
  for (const auto& batch : batches_of(req, trace, opts.batch_size)) {
    json jb;
    std::size_t ev0 = events.size();
    try {
      eng.process_batch(batch);
      jb["rejected"] = false;
    } catch (const BatchRejected& e) {
      jb["rejected"] = true;
      jb["error"] = e.what();
    }
    if (dump) jb["state"] = dump_state(eng);
    if (blob_cb) {
      state_blob(eng, blob);
      blob_cb(bi++, blob.data(), blob.size(), jb["rejected"].get<bool>() ? 1 : 0);
      continue;  // per-batch results go through the callback only
    }
    if (want_events) {
      json je = json::array();
      for (std::size_t i = ev0; i < events.size(); ++i)
        je.push_back({{"t", events[i].time}, {"lane", lane_name(events[i].lane)},
                      {"task", events[i].task}, {"user", events[i].user},
                      {"layer", events[i].layer}});
      jb["events"] = std::move(je);
    }
    batches.push_back(std::move(jb));
  }
  if (!req.value("no_drain", false)) eng.drain();
  if constexpr (std::is_same_v<B, TagBackend>) {
    if (req.value("check_conservation", false)) {
      eng.check_conservation();
      out["conservation"] = "ok";
    }
  }
  if (blob_cb) {
    state_blob(eng, blob);
    blob_cb(~std::uint64_t(0), blob.data(), blob.size(), 0);  // final state, after drain
  } else {
    out["final_state"] = dump_state(eng);
  }
  out["report"] = report_json(eng.report());
  out["batches"] = std::move(batches);
  if constexpr (std::is_same_v<B, ValueBackend>) {
    out["logits"] = logits;
    if (req.value("dump_params", false)) {
      json jp;
      jp["embed"] = params.embed;
      jp["w_out"] = params.w_out;
      json layers = json::array();
      for (const auto& l : params.layers)
        layers.push_back({{"w_in", l.w_in}, {"ln_scale", l.ln_scale},
                          {"w_mlp1", l.w_mlp1}, {"w_mlp2", l.w_mlp2}});
      jp["layers"] = std::move(layers);
      out["params"] = std::move(jp);
    }
    if (req.value("dump_device_kv", false)) {
      // Every resident token's K/V per layer in logical order: the bytes the
      // B200 engine's pool must reproduce (within bf16 rounding).
      json dev = json::object();
      auto& mgr = eng.manager();
      for (UserId u : mgr.known_users()) {
        const SequenceState* s = mgr.find(u);
        json jl = json::array();
        for (std::uint32_t l = 0; l < kv.num_layers; ++l) {
          auto span = eng.device().gather(mgr.user_pages(u), l, s->device_len);
          json toks = json::array();
          for (const auto& e : span) toks.push_back({e.key, e.value});
          jl.push_back(std::move(toks));
        }
        dev[std::to_string(u)] = std::move(jl);
      }
      out["device_kv"] = std::move(dev);
    }
  }
  if (want_events) out["events_jsonl"] = events_to_jsonl(events);
  return out;
}

// Bounded CPU baseline: `threads` independent reference engines (value
// backend, hierarchical mode), each over its own user shard. Warm-up prefill
// (first visit with `history` tokens) is untimed; then every thread replays
// revisits of `delta` new tokens round-robin over its users until `seconds`
// elapse. Returns requests and fresh tokens completed inside the timed window.
json run_bench(const json& req) {
  KVConfig kv = kv_from(req.value("kv", json::object()));
  ModelConfig mc = model_from(req.value("model", json::object()));
  const unsigned threads = req.value("threads", 1u);
  const unsigned users = req.value("users_per_thread", 1u);
  const unsigned history = req.value("history", 1024u);
  const unsigned delta = req.value("delta", 32u);
  const unsigned cands = req.value("candidates", 8u);
  const unsigned batch = req.value("batch_size", 1u);
  const double seconds = req.value("seconds", 10.0);
  ModelParams params = ModelParams::random(mc);
  std::atomic<std::uint64_t> done_req{0}, done_tok{0};
  std::atomic<bool> stop{false};
  std::vector<double> prefill_s(threads, 0.0);
  std::atomic<unsigned> ready{0};
  auto worker = [&](unsigned t) {
    EngineOptions opts;
    opts.mode = Mode::Hierarchical;
    opts.batch_size = batch;
    opts.model = &params;
    Engine<ValueBackend> eng(kv, CostModel{}, opts);
    std::mt19937_64 rng(1000 + t);
    std::uniform_int_distribution<TokenId> tok(0, mc.vocab - 1);
    auto make = [&](UserId u, unsigned dn) {
      Request r;
      r.user = u;
      r.new_tokens.resize(dn);
      for (auto& x : r.new_tokens) x = tok(rng);
      r.candidates.resize(cands);
      for (auto& x : r.candidates) x = tok(rng);
      return r;
    };
    auto t0 = std::chrono::steady_clock::now();
    for (unsigned u = 0; u < users; ++u) eng.process_batch({make(t * users + u, history)});
    prefill_s[t] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    ready.fetch_add(1);
    while (ready.load() < threads) std::this_thread::yield();
    unsigned next = 0;
    while (!stop.load()) {
      std::vector<Request> b;
      for (unsigned i = 0; i < batch; ++i) b.push_back(make(t * users + (next++ % users), delta));
      eng.process_batch(b);
      if (stop.load()) break;  // count only batches finished inside the window
      done_req.fetch_add(b.size());
      done_tok.fetch_add(std::uint64_t(b.size()) * (delta + cands));
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t) pool.emplace_back(worker, t);
  while (ready.load() < threads) std::this_thread::sleep_for(std::chrono::milliseconds(5));
  auto t0 = std::chrono::steady_clock::now();
  std::this_thread::sleep_for(std::chrono::duration<double>(seconds));
  std::uint64_t r = done_req.load(), k = done_tok.load();
  double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  stop.store(true);
  for (auto& th : pool) th.join();
  json out;
  out["requests"] = r;
  out["tokens"] = k;
  out["seconds"] = el;
  out["requests_per_s"] = double(r) / el;
  out["tokens_per_s"] = double(k) / el;
  double mx = 0;
  for (double p : prefill_s) mx = std::max(mx, p);
  out["prefill_s"] = mx;
  return out;
}

json forward(const json& req) {
  ModelParams p = ModelParams::random(model_from(req.value("model", json::object())));
  std::vector<TokenId> hist = req["history"].get<std::vector<TokenId>>();
  std::vector<TokenId> cands = req["candidates"].get<std::vector<TokenId>>();
  std::size_t split = req.value("split", std::size_t(0));
  std::vector<TokenId> prefix(hist.begin(), hist.begin() + std::ptrdiff_t(split));
  std::vector<TokenId> delta(hist.begin() + std::ptrdiff_t(split), hist.end());
  std::vector<LayerKV> cached(p.cfg.num_layers);
  if (split > 0) {
    ForwardOutput warm = forward_full(prefix, {0}, p);
    for (std::uint32_t l = 0; l < p.cfg.num_layers; ++l) cached[l] = warm.new_kv[l].prefix(split);
  }
  ForwardOutput out = forward_incremental(cached, delta, cands, p);
  json j;
  j["logits"] = out.logits;
  j["hidden"] = out.hidden;
  j["ranked"] = rank_candidates(out.logits, cands);
  if (req.value("dump_kv", false)) {
    json layers = json::array();
    for (const auto& kv : out.new_kv) layers.push_back({{"keys", kv.keys}, {"values", kv.values}});
    j["new_kv"] = std::move(layers);
  }
  return j;
}

}  // namespace

extern "C" {

// Returns a malloc'd JSON string; {"error": "..."} on failure. Free with mtkv_ref_free.
char* mtkv_ref_call(const char* request) {
  json out;
  try {
    json req = json::parse(request);
    std::string cmd = req.value("cmd", std::string("run"));
    if (cmd == "gen_trace") {
      out["jsonl"] = trace_to_jsonl(generate_trace(gen_from(req)));
    } else if (cmd == "run") {
      std::vector<Request> trace = trace_from(req["trace"]);
      out = req.value("backend", std::string("tag")) == "value"
                ? run_engine<ValueBackend>(req, trace)
                : run_engine<TagBackend>(req, trace);
    } else if (cmd == "forward") {
      out = forward(req);
    } else if (cmd == "bench") {
      out = run_bench(req);
    } else if (cmd == "footprint") {
      KVConfig kv = kv_from(req.value("kv", json::object()));
      FootprintReport r = memory_footprint(kv, req.value("batch", 16ull), req.value("maxseq", 4096ull),
                                           req.value("residual_mib", 2187ull));
      out = {{"cache_mib", r.cache_mib}, {"uvqk_mib", r.uvqk_mib}, {"output_mib", r.output_mib},
             {"workbench_mib", r.workbench_mib}, {"total_mib", r.total_mib}};
    } else {
      out["error"] = "unknown cmd " + cmd;
    }
  } catch (const std::exception& e) {
    out = json::object();
    out["error"] = e.what();
  }
  std::string s = out.dump();
  char* buf = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return buf;
}

void mtkv_ref_free(char* p) { std::free(p); }

// "run" with the state image of every batch (and of the final, drained state,
// batch = UINT64_MAX) handed to `cb` instead of the JSON state dumps: trace-scale
// runs (thousands of batches, thousands of users) stay cheap to compare.
char* mtkv_ref_run_blobs(const char* request, BlobCb cb) {
  json out;
  try {
    json req = json::parse(request);
    std::vector<Request> trace = trace_from(req["trace"]);
    out = req.value("backend", std::string("tag")) == "value" ? run_engine<ValueBackend>(req, trace, cb)
                                                              : run_engine<TagBackend>(req, trace, cb);
  } catch (const std::exception& e) {
    out = json::object();
    out["error"] = e.what();
  }
  std::string s = out.dump();
  char* buf = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return buf;
}

}  // extern "C"
