// Synthetic request traces with the same RNG streams as the reference
// generator (workload.cpp:85 generate_trace), so a trace produced here on the
// GPU box is byte-for-byte the trace the reference would replay.
// Shape: per-user lifetime length drawn as min + range * U^p (mean-matched),
// visit counts proportional to length, random per-visit split, heavy-tailed
// (lognormal or Pareto) inter-arrival gaps, global stable sort by timestamp.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "workload.hpp"

namespace mtkv_b200 {

static bool gen_ok(const mtkv_gen_config& g, std::string& err) {
  if (g.num_users < 1) err = "gen: need at least one user";
  else if (g.total_requests < 1) err = "gen: need at least one request";
  else if (g.min_len > g.max_len) err = "gen: min_len > max_len";
  else if (g.mean_final_len > double(g.max_len)) err = "gen: infeasible config, mean length exceeds cap";
  else if (g.mean_final_len < double(g.min_len)) err = "gen: mean length below minimum";
  else if (g.candidates < 1) err = "gen: need at least one candidate";
  else if (!(g.gap_log_sigma >= 0 && g.pareto_alpha > 0 && g.pareto_scale_ms > 0))
    err = "gen: distribution parameters out of range";
  return err.empty();
}

int generate(const mtkv_gen_config& g, std::vector<TraceRec>& out, std::string& err) {
  if (!gen_ok(g, err)) return MTKV_ERROR;
  std::mt19937_64 rng(g.seed);
  std::uniform_real_distribution<double> unif(0.0, 1.0);

  const uint32_t U = g.num_users;
  std::vector<uint64_t> life(U);
  double life_sum = 0;
  for (uint32_t u = 0; u < U; ++u) {
    uint64_t len = g.min_len;
    if (g.max_len != g.min_len) {
      const double span = double(g.max_len - g.min_len);
      const double expo = std::max(span / (g.mean_final_len - double(g.min_len)) - 1.0, 1e-9);
      std::uniform_real_distribution<double> u01(0.0, 1.0);
      len = uint64_t(std::llround(double(g.min_len) + span * std::pow(u01(rng), expo)));
    }
    life[u] = len;
    life_sum += double(len);
  }

  std::vector<uint64_t> visits(U);
  uint64_t total = 0;
  for (uint32_t u = 0; u < U; ++u) {
    visits[u] = std::max<uint64_t>(1, uint64_t(std::llround(double(g.total_requests) * double(life[u]) / life_sum)));
    total += visits[u];
  }
  for (uint32_t c = 0; total > g.total_requests; c = (c + 1) % U)
    if (visits[c] > 1) { --visits[c]; --total; }
  for (uint32_t c = 0; total < g.total_requests; c = (c + 1) % U) { ++visits[c]; ++total; }

  const double horizon = std::exp(g.gap_log_mu) * double(g.total_requests) / U * 2.0;
  out.clear();
  out.reserve(g.total_requests);
  for (uint32_t u = 0; u < U; ++u) {
    const uint64_t v = visits[u];
    std::vector<double> w(v);
    double wsum = 0;
    for (auto& x : w) { x = 0.1 + unif(rng); wsum += x; }
    std::vector<uint32_t> dn(v, g.fixed_delta);
    if (g.fixed_delta == 0) {
      uint64_t done = 0;
      double cum = 0;
      for (uint64_t i = 0; i < v; ++i) {
        cum += w[i];
        uint64_t upto = (i + 1 == v) ? life[u] : uint64_t(std::llround(double(life[u]) * cum / wsum));
        upto = std::clamp(upto, done, life[u]);
        dn[i] = uint32_t(upto - done);
        done = upto;
      }
    }
    double t = unif(rng) * horizon;
    for (uint64_t i = 0; i < v; ++i) {
      TraceRec r;
      r.ts = uint64_t(t);
      r.user = u;
      r.dn = dn[i];
      r.nc = g.candidates;
      if (g.vocab > 0) {
        std::uniform_int_distribution<uint32_t> tok(0, g.vocab - 1);
        r.tokens.resize(dn[i]);
        for (auto& x : r.tokens) x = tok(rng);
        r.cands.resize(g.candidates);
        for (auto& x : r.cands) x = tok(rng);
      }
      out.push_back(std::move(r));
      if (!g.pareto) {
        std::normal_distribution<double> z(0.0, 1.0);
        t += std::max(1.0, std::exp(g.gap_log_mu + g.gap_log_sigma * z(rng)));
      } else {
        std::uniform_real_distribution<double> u01(0.0, 1.0);
        const double x = std::max(1e-12, 1.0 - u01(rng));
        t += std::max(1.0, g.pareto_scale_ms * std::pow(x, -1.0 / g.pareto_alpha));
      }
    }
  }
  std::stable_sort(out.begin(), out.end(), [](const TraceRec& a, const TraceRec& b) { return a.ts < b.ts; });
  return MTKV_OK;
}

std::string to_jsonl(const std::vector<TraceRec>& tr) {
  std::string s;
  s.reserve(tr.size() * 48);
  auto arr = [&](const std::vector<uint32_t>& a) {
    s += '[';
    for (size_t i = 0; i < a.size(); ++i) {
      if (i) s += ',';
      s += std::to_string(a[i]);
    }
    s += ']';
  };
  for (const auto& r : tr) {
    s += '{';
    if (!r.tokens.empty() || !r.cands.empty()) { s += "\"cands\":"; arr(r.cands); s += ','; }
    s += "\"dn\":" + std::to_string(r.dn) + ",\"nc\":" + std::to_string(r.nc);
    if (!r.tokens.empty() || !r.cands.empty()) { s += ",\"tokens\":"; arr(r.tokens); }
    s += ",\"ts\":" + std::to_string(r.ts) + ",\"user\":" + std::to_string(r.user) + "}\n";
  }
  return s;
}

}  // namespace mtkv_b200
