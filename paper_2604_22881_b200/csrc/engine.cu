// GPU engine: executes the planner's BatchWork on the B200.
//
// Cross-stream hazards (everything else is ordered on `comp`):
//   1. staging reuse   : H2D of batch i into staging[i%2] waits scatter(i-2)
//   2. host chunk RAW  : H2D of a chunk waits the D2H event of the batch that wrote it
//   3. offload slot    : gather into a reused offload slot waits the previous D2H
// Pages themselves are only touched on `comp` (scatter, append, attention,
// gather), so zero-copy eviction and page reuse need no synchronisation.
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>

namespace mtkv_b200 {

#define CK(x)                                                   \
  do {                                                          \
    cudaError_t e_ = (x);                                       \
    if (e_ != cudaSuccess) {                                    \
      err = std::string(#x) + ": " + cudaGetErrorString(e_);    \
      return MTKV_ERROR;                                        \
    }                                                           \
  } while (0)

int DevBuf::ensure(size_t need, cudaStream_t s) {
  if (need <= bytes) return 0;
  size_t nb = std::max(need, bytes * 2);
  nb = (nb + 255) & ~size_t(255);
  if (s) {
    // stream-ordered: the old buffer is freed after the work already queued on
    // `s` (its only user) and the new one is valid for work queued after this
    // call, so a workspace growing mid-serve stalls nothing
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    bytes = 0;
    if (cudaMallocAsync(&p, nb, s) != cudaSuccess) return -1;
    async = true;
    bytes = nb;
    return 0;
  }
  if (p) {
    cudaDeviceSynchronize();
    cudaFree(p);
  }
  p = nullptr;
  bytes = 0;
  if (cudaMalloc(&p, nb) != cudaSuccess) return -1;
  bytes = nb;
  return 0;
}

void DevBuf::release() {
  if (p) async ? cudaFreeAsync(p, 0) : cudaFree(p);
  p = nullptr;
  bytes = 0;
}

// Candidate scores without the full-vocabulary head (rank_candidates only reads
// the candidates' logits, model.cpp:199): one warp per candidate, the dot of the
// request's last hidden row with the candidate's row of w_out^T (16-B loads).
__global__ void candidate_scores_kernel(float* out, const __nv_bfloat16* x, const __nv_bfloat16* w_out_t,
                                        const uint32_t* last_row, const uint32_t* creq, const uint32_t* cid,
                                        uint32_t n, uint32_t d) {
  const uint32_t j = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (j >= n) return;
  const __nv_bfloat16* xr = x + size_t(last_row[creq[j]]) * d;
  const __nv_bfloat16* wr = w_out_t + size_t(cid[j]) * d;
  float acc = 0.f;
  for (uint32_t k = lane * 8; k < d; k += 256) {
    const uint4 a = *reinterpret_cast<const uint4*>(xr + k), b = *reinterpret_cast<const uint4*>(wr + k);
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 fa = __bfloat1622float2(a2[i]), fb = __bfloat1622float2(b2[i]);
      acc = fmaf(fa.x, fb.x, fmaf(fa.y, fb.y, acc));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[j] = acc;
}

__global__ void pick_scores_kernel(float* out, const float* logits, const uint32_t* creq,
                                   const uint32_t* cid, uint32_t n, uint32_t vocab) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) out[j] = logits[(size_t)creq[j] * vocab + cid[j]];
}

Engine::Engine(const mtkv_kv_config& kv, const mtkv_cost_model& cost, const mtkv_engine_options& opt)
    : planner(kv, cost, opt.mode, opt.backend == MTKV_BACKEND_VALUE), kv_(kv), opt_(opt) {
  value_ = opt.backend == MTKV_BACKEND_VALUE;
  recompute_ = opt.mode == MTKV_MODE_RECOMPUTE;
  g_.L = kv.num_layers;
  g_.H = kv.num_heads;
  g_.D = kv.head_dim;
  g_.d = kv.num_heads * kv.head_dim;
  g_.S = kv.page_size;
  g_.chunk = kv.chunk_size;
  g_.num_pages = recompute_ ? 0 : kv.device_pages;
  chunk_elems_ = size_t(g_.L) * 2 * g_.chunk * g_.d;
  chunk_bytes_ = chunk_elems_ * sizeof(__nv_bfloat16);
  for (int k = 0; k < kRing; ++k) scatter_batch_[k] = d2h_rec_batch_[k] = slot_batch_[k] = -1;
}

Engine::~Engine() {
  if (refill_.joinable()) {
    {
      std::lock_guard<std::mutex> g(slab_mu_);
      stop_refill_ = true;
    }
    slab_cv_.notify_all();
    refill_.join();
  }
  if (comp_) cudaDeviceSynchronize();
  DevBuf* bufs[] = {&trace_, &pool_, &staging_[0], &staging_[1], &offload_, &meta_, &x_, &x2_, &u_, &q_,
                    &mid_, &part_o_, &part_lse_, &logits_, &scores_};
  for (DevBuf* b : bufs) b->release();
  for (void* p : {(void*)w_embed_, (void*)w_in_, (void*)w1_, (void*)w2_, (void*)w_out_, (void*)w_out_t_, (void*)w_ln_})
    if (p) cudaFree(p);
  for (char* s : slabs_) cudaFreeHost(s);
  for (int k = 0; k < kRing; ++k) {
    if (meta_host_[k]) cudaFreeHost(meta_host_[k]);
    if (scores_host_[k]) cudaFreeHost(scores_host_[k]);
    if (logits_host_[k]) cudaFreeHost(logits_host_[k]);
  }
  if (comp_) {
    for (int k = 0; k < kRing; ++k) {
      cudaEventDestroy(ev_onload_[k]); cudaEventDestroy(ev_scatter_[k]);
      cudaEventDestroy(ev_gathered_[k]); cudaEventDestroy(ev_d2h_[k]);
      cudaEventDestroy(ev_done_[k]); cudaEventDestroy(ev_start_[k]); cudaEventDestroy(ev_meta_[k]);
      cudaEventDestroy(ev_stk0_[k]); cudaEventDestroy(ev_stk1_[k]); cudaEventDestroy(ev_h2d0_[k]);
      cudaEventDestroy(ev_h2d1_[k]);
    }
    for (auto e : ev_attn_) cudaEventDestroy(e);
    for (auto e : ev_copy_)
      if (e) cudaEventDestroy(e);
    cudaStreamDestroy(comp_); cudaStreamDestroy(h2d_); cudaStreamDestroy(d2h_);
  }
}

// Reference weight init (model.cpp:34): mt19937_64(seed), N(0, 0.3/sqrt(d)) per
// matrix in the order embed, per layer (w_in, ln_scale ~ N(0,1), w_mlp1, w_mlp2),
// w_out; rounded to bf16 for the tensor cores (ln_scale kept fp32).
void Engine::init_weights() {
  const auto& mc = opt_.model;
  const size_t d = g_.d, V = mc.vocab, L = g_.L;
  std::mt19937_64 rng(mc.seed);
  const double s = 0.3 / std::sqrt(double(d));
  auto draw = [&](size_t n, double sd) {
    std::normal_distribution<double> dist(0.0, sd);
    std::vector<double> m(n);
    for (auto& v : m) v = dist(rng);
    return m;
  };
  auto to_bf16 = [](const std::vector<double>& m, std::vector<__nv_bfloat16>& out, size_t at) {
    for (size_t i = 0; i < m.size(); ++i) out[at + i] = __float2bfloat16(float(m[i]));
  };
  std::vector<__nv_bfloat16> embed(V * d), w_in(L * d * 4 * d), w1(L * d * d), w2(L * d * d), w_out(d * V);
  std::vector<float> ln(L * d);
  to_bf16(draw(V * d, s), embed, 0);
  for (size_t l = 0; l < L; ++l) {
    to_bf16(draw(d * 4 * d, s), w_in, l * d * 4 * d);
    auto lv = draw(d, 1.0);
    for (size_t i = 0; i < d; ++i) ln[l * d + i] = float(lv[i]);
    to_bf16(draw(d * d, s), w1, l * d * d);
    to_bf16(draw(d * d, s), w2, l * d * d);
  }
  to_bf16(draw(d * V, s), w_out, 0);
  auto up = [](auto& host, auto** dev) {
    cudaMalloc((void**)dev, host.size() * sizeof(host[0]));
    cudaMemcpy(*dev, host.data(), host.size() * sizeof(host[0]), cudaMemcpyHostToDevice);
  };
  up(embed, &w_embed_);
  up(w_in, &w_in_);
  up(w1, &w1_);
  up(w2, &w2_);
  up(w_out, &w_out_);
  // w_out^T [V x d] for the candidate-score kernel (one contiguous row per candidate)
  if (d % 8 == 0) {
    std::vector<__nv_bfloat16> wt(V * d);
    for (size_t k = 0; k < d; ++k)
      for (size_t v = 0; v < V; ++v) wt[v * d + k] = w_out[k * V + v];
    up(wt, &w_out_t_);
  }
  up(ln, &w_ln_);
}

int Engine::init(std::string& err) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    err = "no CUDA device available (the B200 engine has no CPU fallback)";
    return MTKV_NO_DEVICE;
  }
  if (opt_.device < 0 || opt_.device >= ndev) {
    err = "invalid CUDA device ordinal";
    return MTKV_NO_DEVICE;
  }
  CK(cudaSetDevice(opt_.device));
  if (g_.d % 2 != 0 || g_.d > 512) {
    err = "engine: hidden width H*D must be even and <= 512";
    return MTKV_ERROR;
  }
  if (g_.D > 128) {
    err = "engine: head_dim must be <= 128";
    return MTKV_ERROR;
  }
  if (kv_.bytes_per_element != 2) {
    err = "engine: the device pool stores bf16 (bytes_per_element must be 2)";
    return MTKV_ERROR;
  }
  // tcgen05 attention for every production shape: the two-lane kernel for
  // head_dim 64/128, the column-split one for head_dim 32; the mma.sync kernel
  // covers the reference's tiny test models (attn_kind: MTKV_ATTN=mma|tc1 force
  // the others for A/B measurements)
  attn_kind_ = attn_kind(g_);
  use_tc_ = attn_kind_ != AttnKind::Mma;
  n_sm_ = num_sms();
  CK(cudaStreamCreateWithFlags(&comp_, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));
  for (int k = 0; k < kRing; ++k) {
    CK(cudaEventCreateWithFlags(&ev_onload_[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_scatter_[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_gathered_[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_d2h_[k], cudaEventDisableTiming));
    CK(cudaEventCreate(&ev_done_[k]));
    CK(cudaEventCreate(&ev_start_[k]));
    CK(cudaEventCreateWithFlags(&ev_meta_[k], cudaEventDisableTiming));
    CK(cudaEventCreate(&ev_stk0_[k]));
    CK(cudaEventCreate(&ev_stk1_[k]));
    CK(cudaEventCreate(&ev_h2d0_[k]));
    CK(cudaEventCreate(&ev_h2d1_[k]));
  }
  if (!recompute_) {
    if (pool_.ensure(size_t(g_.L) * g_.num_pages * 2 * g_.S * g_.d * sizeof(__nv_bfloat16))) {
      err = "engine: cannot allocate the device page pool";
      return MTKV_ERROR;
    }
    CK(cudaMemset(pool_.p, 0, pool_.bytes));
  }
  const uint64_t slots = std::max<uint64_t>(1, kv_.offload_quota / kv_.chunk_size);
  if (!recompute_ && opt_.mode == MTKV_MODE_HIERARCHICAL) {
    if (offload_.ensure(slots * chunk_bytes_)) {
      err = "engine: cannot allocate the offload buffer";
      return MTKV_ERROR;
    }
    off_free_.clear();
    for (uint64_t s = slots; s-- > 0;) off_free_.push_back(uint32_t(s));
    off_slot_batch_.assign(slots, -1);
  }
  // host extents of ~8 MB (>= 1 chunk) and slabs of >= 4 extents
  const size_t extent_bytes = size_t(opt_.host_extent_mb ? opt_.host_extent_mb : 8) << 20;
  chunks_per_extent_ = uint32_t(std::max<size_t>(1, extent_bytes / chunk_bytes_));
  slab_bytes_ = std::max<size_t>(size_t(64) << 20, chunk_bytes_ * chunks_per_extent_ * 4);
  if (opt_.mode == MTKV_MODE_HIERARCHICAL) {
    // reserve the expected host store now: cudaHostAlloc takes the driver lock
    // and would stall launches if it ran while serving
    const size_t want = size_t(opt_.host_reserve_mb) << 20;
    for (size_t got = 0; got < want; got += slab_bytes_) {
      char* s = nullptr;
      CK(cudaHostAlloc((void**)&s, slab_bytes_, cudaHostAllocDefault));
      slabs_.push_back(s);
      spare_slabs_.push_back(s);
    }
    refill_ = std::thread([this] { slab_refill_loop(); });
  }
  // staging for the largest onload a batch may plan (KVConfig::onload_pages),
  // allocated up front so no timed batch reallocates (capped; grows lazily past it)
  if (opt_.mode == MTKV_MODE_HIERARCHICAL) {
    const size_t slots = size_t(kv_.onload_pages) * kv_.page_size / kv_.chunk_size;
    const size_t bytes = std::min(slots * chunk_bytes_, size_t(8) << 30);
    if (bytes && (staging_[0].ensure(bytes) || staging_[1].ensure(bytes))) {
      err = "engine: cannot allocate the onload staging buffers";
      return MTKV_ERROR;
    }
  }
  if (value_) init_weights();
  if (set_onload_policy(opt_.onload_policy, opt_.onload_gbs, opt_.recompute_mtok_s, err)) return MTKV_ERROR;
  if (opt_.device_planner) {
    if (recompute_) {
      err = "engine: the device planner needs a cached mode (gpu_only or hierarchical)";
      return MTKV_ERROR;
    }
    const uint32_t max_users = opt_.max_users ? opt_.max_users : 65536;
    const uint32_t max_pages = opt_.max_user_pages ? opt_.max_user_pages : kv_.device_pages;
    if (uint64_t(max_users) * max_pages > (uint64_t(1) << 30)) {
      err = "engine: device planner page table too large (set max_users / max_user_pages)";
      return MTKV_ERROR;
    }
    if (ctl_.init(kv_.device_pages, kv_.page_size, kv_.chunk_size, opt_.mode == MTKV_MODE_HIERARCHICAL, max_users,
                  max_pages, uint64_t(kv_.onload_pages) * kv_.page_size, err))
      return MTKV_ERROR;
    planner.set_device_ctl(&ctl_);
  }
  CK(cudaGetLastError());
  return MTKV_OK;
}

// Pinned host store. A user's chunks live in per-user extents of
// chunks_per_extent_ consecutive chunks, so the onload of a user's persisted
// prefix is a handful of large copy-engine transfers instead of one per chunk.
// Extents are carved from pinned slabs; a background thread keeps spare slabs
// ready so cudaHostAlloc never lands on the serving path.
char* Engine::take_slab() {
  {
    std::lock_guard<std::mutex> g(slab_mu_);
    if (!spare_slabs_.empty()) {
      char* s = spare_slabs_.back();
      spare_slabs_.pop_back();
      slab_cv_.notify_one();
      return s;
    }
  }
  char* s = nullptr;
  if (cudaHostAlloc((void**)&s, slab_bytes_, cudaHostAllocDefault) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> g(slab_mu_);
  slabs_.push_back(s);
  slab_cv_.notify_one();
  return s;
}

void Engine::slab_refill_loop() {
  cudaSetDevice(opt_.device);
  std::unique_lock<std::mutex> lk(slab_mu_);
  while (!stop_refill_) {
    if (spare_slabs_.size() < kSpareSlabs) {
      lk.unlock();
      char* s = nullptr;
      const bool ok = cudaHostAlloc((void**)&s, slab_bytes_, cudaHostAllocDefault) == cudaSuccess;
      lk.lock();
      if (!ok) break;
      slabs_.push_back(s);
      spare_slabs_.push_back(s);
      continue;
    }
    slab_cv_.wait(lk, [&] { return stop_refill_ || spare_slabs_.size() < kSpareSlabs; });
  }
}

int Engine::host_chunk(uint64_t id, uint32_t user, uint32_t index, std::string& err) {
  if (id < chunk_ptr_.size() && chunk_ptr_[id]) return MTKV_OK;
  std::vector<char*>& ext = user_extents_[user];
  const uint32_t e = index / chunks_per_extent_;
  while (ext.size() <= e) {
    const size_t eb = chunk_bytes_ * chunks_per_extent_;
    if (!cur_slab_ || slab_used_ + eb > slab_bytes_) {
      cur_slab_ = take_slab();
      slab_used_ = 0;
      if (!cur_slab_) {
        err = "engine: pinned host allocation failed";
        return MTKV_ERROR;
      }
    }
    ext.push_back(cur_slab_ + slab_used_);
    slab_used_ += eb;
  }
  if (chunk_ptr_.size() <= id) {
    const size_t n = std::max<size_t>(id + 1, chunk_ptr_.size() * 2);
    chunk_ptr_.resize(n, nullptr);
    chunk_d2h_batch_.resize(n, -1);
    chunk_off_slot_.resize(n, -1);
  }
  chunk_ptr_[id] = ext[e] + size_t(index % chunks_per_extent_) * chunk_bytes_;
  return MTKV_OK;
}

static size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <class T>
static T* carve(char* base, size_t& off, size_t count) {
  T* p = reinterpret_cast<T*>(base + off);
  off = align16(off + count * sizeof(T));
  return p;
}

// dense layers: tcgen05 kernel (gemm_tc.cu) for every shape it covers, mma.sync
// otherwise; MTKV_GEMM=mma forces the legacy kernel for A/B measurements
int Engine::gemm(const GemmArgs& a, uint64_t a_rows_alloc, std::string& err) {
  static const bool force_mma = [] {
    const char* f = std::getenv("MTKV_GEMM");
    return f && std::string(f) == "mma";
  }();
  if (!force_mma && gemm_tc_supported(a)) {
    if (launch_gemm_tc(a, a_rows_alloc, comp_)) {
      err = "engine: cuTensorMapEncodeTiled (GEMM operands) failed";
      return MTKV_ERROR;
    }
  } else {
    launch_gemm(a, comp_);
  }
  return MTKV_OK;
}

// Value backend: the payload is validated before the planner touches any state
// (a batch that fails here leaves the engine exactly as it was). The messages
// are the reference model's (model.cpp:159, :162; manager.cpp:103).
int Engine::validate_payload(const mtkv_request* reqs, uint32_t n, std::string& err) const {
  const uint32_t V = opt_.model.vocab;
  for (uint32_t i = 0; i < n; ++i) {
    const mtkv_request& r = reqs[i];
    if (r.candidate_count < 1) { err = "request: need at least one candidate"; return MTKV_ERROR; }
    if ((r.new_token_count && !r.new_tokens) || !r.candidates) {
      err = "value mode: trace must carry explicit token ids";
      return MTKV_ERROR;
    }
    for (uint32_t j = 0; j < r.new_token_count; ++j)
      if (r.new_tokens[j] >= V) { err = "forward: token id out of vocabulary"; return MTKV_ERROR; }
    for (uint32_t j = 0; j < r.candidate_count; ++j)
      if (r.candidates[j] >= V) { err = "forward: token id out of vocabulary"; return MTKV_ERROR; }
  }
  return MTKV_OK;
}

// Executor policy for host hits (mtkv_engine_options::onload_policy); may change
// between batches (the control plane does not depend on it).
int Engine::set_onload_policy(uint32_t policy, double gbs, double mtok_s, std::string& err) {
  if (policy > MTKV_ONLOAD_ADAPTIVE) {
    err = "engine: unknown onload_policy";
    return MTKV_ERROR;
  }
  opt_.onload_policy = policy;
  opt_.onload_gbs = gbs;
  opt_.recompute_mtok_s = mtok_s;
  // default re-encode rate: the layer stack's FLOPs per token (dense 12 d^2 plus
  // attention over ~2K keys) at ~200 TFLOP/s effective (measured 38 M tok/s for
  // 4K-token histories at L=4, d=256)
  const double d = g_.d, flops = double(g_.L) * (12.0 * d * d + 2.0 * 2.0 * 2048.0 * d);
  const double tps = mtok_s > 0 ? mtok_s * 1e6 : 2e14 / flops;
  planner.set_onload_policy(int(policy), (gbs > 0 ? gbs : 54.0) * 1e9, tps);
  // no rate given: the value engine measures both (calibrate_from) and the
  // policy follows the measured rates; the tag backend has no layer stack to time
  calibrate_ = value_ && policy == MTKV_ONLOAD_ADAPTIVE && mtok_s <= 0;
  cal_tps_ = cal_Bps_ = 0;
  for (int k = 0; k < kRing; ++k) cal_rows_[k] = cal_bytes_[k] = 0;
  return MTKV_OK;
}

// Adaptive policy calibration from a completed batch (ring slot k): the layer
// stack's rows per second on the SMs and the onload bytes per second over the
// host link, as exponential moving averages. The policy balances the two per
// batch, so its rates must be this box's, not a model's: at d = 256 the stack
// runs ~2.5x faster than the FLOP estimate (its attention is softmax-bound,
// not FLOP-bound). Changes only which host hits are re-encoded instead of
// onloaded; the control plane never sees it.
void Engine::calibrate_from(int k) {
  if (!calibrate_) return;
  constexpr double a = 0.25;
  float ms = 0;
  if (cal_rows_[k] >= 4096 && cudaEventElapsedTime(&ms, ev_stk0_[k], ev_stk1_[k]) == cudaSuccess && ms > 0) {
    const double tps = double(cal_rows_[k]) / (ms * 1e-3);
    cal_tps_ = cal_tps_ > 0 ? (1 - a) * cal_tps_ + a * tps : tps;
  }
  if (cal_bytes_[k] >= (size_t(8) << 20) && cudaEventElapsedTime(&ms, ev_h2d0_[k], ev_h2d1_[k]) == cudaSuccess && ms > 0) {
    const double bps = double(cal_bytes_[k]) / (ms * 1e-3);
    cal_Bps_ = cal_Bps_ > 0 ? (1 - a) * cal_Bps_ + a * bps : bps;
  }
  cal_rows_[k] = cal_bytes_[k] = 0;
  (void)cudaGetLastError();  // an unavailable timing is skipped, not an engine error
  // MTKV_ADAPTIVE_SM_BIAS (A/B knob): scales the measured layer-stack rate
  // before the split (its event bracket also spans waits on onloads)
  static const double bias = [] {
    const char* e = std::getenv("MTKV_ADAPTIVE_SM_BIAS");
    const double v = e ? std::atof(e) : 1.0;
    return v > 0.25 && v < 4.0 ? v : 1.0;
  }();
  if (cal_tps_ > 0 && cal_Bps_ > 0) planner.set_onload_policy(int(opt_.onload_policy), cal_Bps_, cal_tps_ * bias);
}

int Engine::process_batch(const mtkv_request* reqs, uint32_t n, std::string& err) {
  CK(cudaSetDevice(opt_.device));
  if (value_ && validate_payload(reqs, n, err)) return MTKV_ERROR;
  BatchWork w;
  const auto t0 = std::chrono::steady_clock::now();
  planner.plan_batch(reqs, n, w);
  last_plan_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  const int rc = enqueue(w, reqs, n, err);
  if (w.rc) {
    err = w.error;
    planner.keep_last(w);
    return w.rc;
  }
  planner.keep_last(w);
  return rc;
}

int Engine::enqueue(const BatchWork& w, const mtkv_request* reqs, uint32_t n, std::string& err) {
  // completions that fired at batch start free their offload slots
  for (uint64_t id : w.persisted) {
    if (id < chunk_off_slot_.size() && chunk_off_slot_[id] >= 0) {
      off_free_.push_back(uint32_t(chunk_off_slot_[id]));
      chunk_off_slot_[id] = -1;
    }
  }
  if (w.rc || n == 0) return MTKV_OK;
  const int k = int(batch_no_ % kRing);
  if (batch_no_ >= kRing) {  // ring slot free: the batch leaving it is complete, its offload D2H included
    CK(cudaEventSynchronize(ev_done_[k]));
    if (d2h_rec_batch_[k] >= 0) CK(cudaEventSynchronize(ev_d2h_[k]));
    d2h_done_upto_ = int64_t(batch_no_) - kRing;
    calibrate_from(k);
  }

  const uint32_t S = g_.S, d = g_.d, H = g_.H, V = value_ ? opt_.model.vocab : 0;

  // ---- recompute mode: transient pages for every fresh row ----
  std::vector<uint32_t> tpages;
  std::vector<uint32_t> t_off(n), t_np(n), t_soff(n), t_ns(n);
  if (recompute_) {
    uint32_t next = 0;
    for (uint32_t r = 0; r < n; ++r) {
      const auto& R = w.reqs[r];
      t_off[r] = uint32_t(tpages.size());
      t_np[r] = (R.n_hist + S - 1) / S;
      for (uint32_t i = 0; i < t_np[r]; ++i) tpages.push_back(next++);
      t_soff[r] = uint32_t(tpages.size());
      t_ns[r] = (R.plan.num_candidates + S - 1) / S;
      for (uint32_t i = 0; i < t_ns[r]; ++i) tpages.push_back(next++);
    }
    if (next > g_.num_pages) {
      g_.num_pages = std::max<uint32_t>(next, g_.num_pages * 2);
      if (pool_.ensure(size_t(g_.L) * g_.num_pages * 2 * S * d * sizeof(__nv_bfloat16), comp_)) {
        err = "engine: cannot grow the transient page pool";
        return MTKV_ERROR;
      }
      // fresh allocation bits may be NaN patterns: page padding and unused
      // candidate slots are read with P = 0, and 0 x NaN poisons O
      CK(cudaMemsetAsync(pool_.p, 0, pool_.bytes, comp_));
    }
  }
  const std::vector<uint32_t>& pages = recompute_ ? tpages : w.pages;

  // ---- rows, attention work, metadata sizes ----
  // device requests: the batch's requests, then one extra per split host hit
  // (the re-encoded head of its prefix, positions [0, head_rows), no
  // candidates) — after the batch's requests so result rows stay in request order
  uint32_t n_extra = 0;
  for (uint32_t r = 0; r < n; ++r) n_extra += w.reqs[r].head_rows ? 1 : 0;
  const uint32_t nr = n + n_extra;
  std::vector<ReqDev> rd(nr);
  std::vector<uint32_t> rd_tok(nr);  // offset of each device request's token ids in w.tokens
  uint32_t rows = 0, max_hist = 0, ncand_total = 0;
  const bool tc = use_tc_;
  for (uint32_t r = 0; r < n; ++r) {
    const ReqWork& R = w.reqs[r];
    ReqDev& x = rd[r];
    x = ReqDev{};
    x.q_row0 = rows;
    x.n_hist = R.n_hist;
    x.n_cand = R.plan.num_candidates;
    x.n_q = x.n_hist + x.n_cand;
    x.start = R.start;
    x.pages_off = recompute_ ? t_off[r] : R.pages_off;
    x.n_pages = recompute_ ? t_np[r] : R.n_pages;
    x.scratch_off = recompute_ ? t_soff[r] : R.scratch_off;
    x.n_scratch = recompute_ ? t_ns[r] : R.n_scratch;
    x.user = R.plan.user;
    // keys from dep_start on are appended by this batch's projection GEMM: its
    // own rows, a split host hit's re-encoded head (from 0), or an earlier
    // occurrence of the user in the batch
    x.dep_start = R.head_rows ? 0 : x.start;
    for (uint32_t q = 0; q < r; ++q)
      if (w.reqs[q].slot == R.slot) {
        x.dep_start = std::min(x.dep_start, rd[q].dep_start);
        break;
      }
    rd_tok[r] = R.tok_off;
    rows += x.n_q;
    ncand_total += x.n_cand;
    max_hist = std::max(max_hist, x.n_hist);
  }
  for (uint32_t r = 0, e = n; r < n; ++r) {
    const ReqWork& R = w.reqs[r];
    if (!R.head_rows) continue;
    ReqDev& x = rd[e];
    x = ReqDev{};
    x.q_row0 = rows;
    x.n_hist = x.n_q = R.head_rows;
    x.start = 0;
    x.pages_off = R.pages_off;
    x.n_pages = R.n_pages;
    x.user = R.plan.user;
    x.dep_start = 0;
    rd_tok[e] = R.head_tok_off;
    rows += x.n_q;
    max_hist = std::max(max_hist, x.n_hist);
    ++e;
  }
  last_rows_ = rows;
  if (value_) {
    plan_attention(rd.data(), nr, g_, tc, attn_plan_ctas(attn_kind_, n_sm_), plan_,
                   attn_kind_ == AttnKind::Tc && attn_pair_wanted(g_, rd.data(), nr));
    if (attn_kind_ == AttnKind::Pp && plan_.n_ctas() % 2) plan_.cta_off.push_back(plan_.cta_off.back());
  }
  // Last layer: the head reads only each request's last row (model.cpp:195
  // logits = e[last] W_out), so after the projection GEMM (which still appends
  // every fresh row's K/V of that layer) the attention, gate/norm and MLP run
  // for one row per request — none for a split host hit's re-encoded head.
  // rd_last: the requests with q_skip = n_q - 1; rd_gate: the same segments seen
  // from compact rows (row r = request r).
  static const bool full_last = [] {  // MTKV_LAST_LAYER=full: every row through the last layer (A/B switch)
    const char* e = std::getenv("MTKV_LAST_LAYER");
    return e && e[0] == 'f';
  }();
  // (small batches are host-bound: the second attention plan costs more than
  // the last layer's few rows; measured ~2.5 % on configs[0])
  const bool reduce_last = value_ && attn_kind_ == AttnKind::Tc && !full_last && rows >= 4096;
  std::vector<ReqDev> rd_last, rd_gate;
  if (reduce_last) {
    rd_last.assign(rd.begin(), rd.begin() + n);
    for (ReqDev& x : rd_last) x.q_skip = x.n_q - 1;
    plan_attention(rd_last.data(), n, g_, tc, attn_plan_ctas(attn_kind_, n_sm_), plan_last_);
    rd_gate = rd_last;
    for (uint32_t r = 0; r < n; ++r) {
      rd_gate[r].q_row0 = r;
      rd_gate[r].n_q = 1;
    }
  }
  const uint32_t n_segs_l = reduce_last ? uint32_t(plan_last_.segs.size()) : 0;
  const uint32_t n_items_l = reduce_last ? plan_last_.n_ctas() : 0;
  const uint32_t n_pieces_l = reduce_last ? uint32_t(plan_last_.pieces.size()) : 0;
  const uint32_t bq = plan_.bm;
  const uint32_t n_segs = value_ ? uint32_t(plan_.segs.size()) : 0;
  const uint32_t n_items = value_ ? (tc ? plan_.n_ctas() : uint32_t(plan_.items.size())) : 0;
  const uint32_t n_pieces = value_ && tc ? uint32_t(plan_.pieces.size()) : 0;
  const uint32_t n_on = uint32_t(w.onloads.size()), n_off = uint32_t(w.offloads.size());
  uint32_t n_gblk = 0;  // gate/norm row blocks
  if (value_)
    for (uint32_t r = 0; r < nr; ++r) n_gblk += (rd[r].n_q + kGateBlockRows - 1) / kGateBlockRows;

  size_t need = 0;
  need = align16(need + nr * sizeof(ReqDev));
  need = align16(need + pages.size() * sizeof(uint32_t));
  need = align16(need + rows * sizeof(uint32_t));      // tok
  need = align16(need + rows * sizeof(uint64_t));      // kv_off
  need = align16(need + rows * sizeof(uint32_t));      // row_req
  need = align16(need + nr * sizeof(uint32_t));        // last_row
  need = align16(need + n_segs * sizeof(AttnSeg));
  need = align16(need + (tc ? 0 : n_items) * sizeof(AttnItem));
  need = align16(need + n_pieces * sizeof(AttnPiece));
  need = align16(need + (tc ? n_items + 1 : 0) * sizeof(uint32_t));
  need = align16(need + (n_on + n_off) * sizeof(ChunkWork));
  need = align16(need + 2 * ncand_total * sizeof(uint32_t));
  need = align16(need + 2 * n_gblk * sizeof(uint32_t));
  if (reduce_last) {
    need = align16(need + n * sizeof(ReqDev));              // rd_last
    need = align16(need + n * sizeof(ReqDev));              // rd_gate
    need = align16(need + n_segs_l * sizeof(AttnSeg));
    need = align16(need + n_pieces_l * sizeof(AttnPiece));
    need = align16(need + (n_items_l + 1) * sizeof(uint32_t));
    need = align16(need + 2 * n * sizeof(uint32_t));        // identity rows, u rows
  }
  if (meta_host_bytes_[k] < need) {
    if (meta_host_[k]) cudaFreeHost(meta_host_[k]);
    meta_host_bytes_[k] = std::max(need, meta_host_bytes_[k] * 2);
    CK(cudaHostAlloc((void**)&meta_host_[k], meta_host_bytes_[k], cudaHostAllocDefault));
  }
  // one 256-B aligned device slot per ring entry (kernels read 16-B vectors from it)
  if (need > meta_slot_) {
    meta_slot_ = (std::max(need, 2 * meta_slot_) + 255) & ~size_t(255);
    if (meta_.ensure(meta_slot_ * kRing)) { err = "engine: metadata alloc"; return MTKV_ERROR; }
  }
  char* hb = meta_host_[k];
  char* db = static_cast<char*>(meta_.p) + size_t(k) * meta_slot_;
  size_t off = 0;
  ReqDev* h_req = carve<ReqDev>(hb, off, nr);
  const size_t o_pages = off;
  uint32_t* h_pages = carve<uint32_t>(hb, off, pages.size());
  const size_t o_tok = off;
  uint32_t* h_tok = carve<uint32_t>(hb, off, rows);
  const size_t o_kv = off;
  uint64_t* h_kv = carve<uint64_t>(hb, off, rows);
  const size_t o_rr = off;
  uint32_t* h_rr = carve<uint32_t>(hb, off, rows);
  const size_t o_last = off;
  uint32_t* h_last = carve<uint32_t>(hb, off, nr);
  const size_t o_segs = off;
  AttnSeg* h_segs = carve<AttnSeg>(hb, off, n_segs);
  const size_t o_items = off;
  AttnItem* h_items = carve<AttnItem>(hb, off, tc ? 0 : n_items);
  const size_t o_pieces = off;
  AttnPiece* h_pieces = carve<AttnPiece>(hb, off, n_pieces);
  const size_t o_ctaoff = off;
  uint32_t* h_ctaoff = carve<uint32_t>(hb, off, tc ? n_items + 1 : 0);
  const size_t o_chunks = off;
  ChunkWork* h_chunks = carve<ChunkWork>(hb, off, n_on + n_off);
  const size_t o_cand = off;
  uint32_t* h_creq = carve<uint32_t>(hb, off, ncand_total);
  uint32_t* h_cid = h_creq + ncand_total;
  off = align16(o_cand + 2 * ncand_total * sizeof(uint32_t));
  const size_t o_gblk = off;
  uint32_t* h_gblk = carve<uint32_t>(hb, off, 2 * n_gblk);
  for (uint32_t r = 0, b = 0; r < nr && value_; ++r)
    for (uint32_t i0 = 0; i0 < rd[r].n_q; i0 += kGateBlockRows, ++b) {
      h_gblk[2 * b] = r;
      h_gblk[2 * b + 1] = i0;
    }

  size_t o_req_l = 0, o_req_g = 0, o_segs_l = 0, o_pieces_l = 0, o_ctaoff_l = 0, o_rowc = 0;
  if (reduce_last) {
    o_req_l = off;
    std::memcpy(carve<ReqDev>(hb, off, n), rd_last.data(), n * sizeof(ReqDev));
    o_req_g = off;
    std::memcpy(carve<ReqDev>(hb, off, n), rd_gate.data(), n * sizeof(ReqDev));
    o_segs_l = off;
    std::memcpy(carve<AttnSeg>(hb, off, n_segs_l), plan_last_.segs.data(), n_segs_l * sizeof(AttnSeg));
    o_pieces_l = off;
    std::memcpy(carve<AttnPiece>(hb, off, n_pieces_l), plan_last_.pieces.data(), n_pieces_l * sizeof(AttnPiece));
    o_ctaoff_l = off;
    std::memcpy(carve<uint32_t>(hb, off, n_items_l + 1), plan_last_.cta_off.data(), (n_items_l + 1) * sizeof(uint32_t));
    o_rowc = off;
    uint32_t* rowc = carve<uint32_t>(hb, off, 2 * n);  // [0, n): identity; [n, 2n): each request's last batch row
    for (uint32_t r = 0; r < n; ++r) {
      rowc[r] = r;
      rowc[n + r] = rd[r].q_row0 + rd[r].n_q - 1;
    }
  }
  if (off > need) { err = "engine: metadata layout overflow"; return MTKV_ERROR; }  // carve order == need order
  std::memcpy(h_req, rd.data(), nr * sizeof(ReqDev));
  if (!pages.empty()) std::memcpy(h_pages, pages.data(), pages.size() * sizeof(uint32_t));
  std::vector<uint32_t>& cands_k = slot_cands_[k];
  std::vector<uint32_t>& nc_k = slot_nc_[k];
  cands_k.clear();
  nc_k.assign(n, 0);
  slot_batch_[k] = int64_t(batch_no_);
  uint32_t cj = 0;
  if (n_segs) std::memcpy(h_segs, plan_.segs.data(), n_segs * sizeof(AttnSeg));
  if (!tc && n_items) std::memcpy(h_items, plan_.items.data(), n_items * sizeof(AttnItem));
  if (n_pieces) std::memcpy(h_pieces, plan_.pieces.data(), n_pieces * sizeof(AttnPiece));
  if (tc && n_items) std::memcpy(h_ctaoff, plan_.cta_off.data(), (n_items + 1) * sizeof(uint32_t));
  for (uint32_t r = 0; r < nr; ++r) {
    const ReqDev& x = rd[r];
    // per-row metadata, page by page (re-encoded prefixes make batches of ~1e5
    // rows: one division per page, not per row)
    std::fill(h_rr + x.q_row0, h_rr + x.q_row0 + x.n_q, r);
    if (value_) std::memcpy(h_tok + x.q_row0, w.tokens.data() + rd_tok[r], size_t(x.n_q) * sizeof(uint32_t));
    else std::fill(h_tok + x.q_row0, h_tok + x.q_row0 + x.n_q, 0u);
    for (uint32_t i = 0; i < x.n_hist;) {  // history rows: positions start + i of the user's pages
      const uint64_t pos = x.start + i;
      const uint32_t slot0 = uint32_t(pos % S), take = std::min<uint32_t>(S - slot0, x.n_hist - i);
      const uint64_t base = uint64_t(pages[x.pages_off + uint32_t(pos / S)]) * 2 * S;
      for (uint32_t j = 0; j < take; ++j) h_kv[x.q_row0 + i + j] = (base + slot0 + j) * d;
      i += take;
    }
    for (uint32_t c = 0; c < x.n_cand; ++c)  // candidate rows: the request's scratch pages
      h_kv[x.q_row0 + x.n_hist + c] = (uint64_t(pages[x.scratch_off + c / S]) * 2 * S + c % S) * d;
    h_last[r] = x.q_row0 + x.n_q - 1;
    if (r >= n) continue;  // an extra (re-encoded head) has no candidates
    nc_k[r] = x.n_cand;
    for (uint32_t c = 0; c < x.n_cand; ++c) {
      const uint32_t id = value_ ? w.tokens[rd_tok[r] + x.n_hist + c] : 0;
      h_creq[cj] = r;
      h_cid[cj] = id;
      cands_k.push_back(id);
      ++cj;
    }
  }
  for (uint32_t j = 0; j < n_on; ++j) h_chunks[j] = ChunkWork{j, w.onloads[j].pages_off};
  std::vector<uint32_t> off_slots(n_off);
  for (uint32_t j = 0; j < n_off; ++j) {
    if (off_free_.empty()) { err = "engine: offload slots exhausted (quota accounting broken)"; return MTKV_ERROR; }
    off_slots[j] = off_free_.back();
    off_free_.pop_back();
    h_chunks[n_on + j] = ChunkWork{off_slots[j], w.offloads[j].pages_off};
  }

  // ---- batch metadata: on the h2d stream, ahead of this batch's chunk copies.
  // (Issued on comp it shares the H2D copy engine's queue with the chunk copies
  // and, waiting for comp to reach it, held the next batch's onload back until
  // this batch's scatter had run: measured ~200 us copy-engine idle per batch.)
  CK(cudaMemcpyAsync(db, hb, off, cudaMemcpyHostToDevice, h2d_));
  CK(cudaEventRecord(ev_meta_[k], h2d_));
  h2d_bytes_ += off;

  // ---- onload: copy-engine H2D into staging[batch % 2] ----
  const int sb = int(batch_no_ % 2);
  if (n_on) {
    if (staging_[sb].bytes < size_t(n_on) * chunk_bytes_ &&
        staging_[sb].ensure(size_t(n_on) * chunk_bytes_)) {
      err = "engine: staging alloc";
      return MTKV_ERROR;
    }
    if (batch_no_ >= 2) CK(cudaStreamWaitEvent(h2d_, ev_scatter_[(batch_no_ - 2) % kRing], 0));
    if (calibrate_) {
      CK(cudaEventRecord(ev_h2d0_[k], h2d_));
      cal_bytes_[k] = uint64_t(n_on) * chunk_bytes_;
    }
    int64_t waited = -1;
    for (uint32_t j = 0; j < n_on;) {
      // a run of chunks contiguous in the host extent -> one transfer into
      // consecutive staging slots
      uint32_t run = 1;
      const ChunkMove& m = w.onloads[j];
      if (m.chunk_id >= chunk_ptr_.size() || !chunk_ptr_[m.chunk_id]) {
        err = "engine: onload of a chunk with no host copy";
        return MTKV_ERROR;
      }
      int64_t b = chunk_d2h_batch_[m.chunk_id];
      while (j + run < n_on) {
        // same user, next chunk, same extent (one pinned allocation per copy)
        const ChunkMove& nx = w.onloads[j + run];
        if (nx.user != m.user || nx.chunk_index != m.chunk_index + run ||
            nx.chunk_index / chunks_per_extent_ != m.chunk_index / chunks_per_extent_ ||
            nx.chunk_id >= chunk_ptr_.size() || chunk_ptr_[nx.chunk_id] != chunk_ptr_[m.chunk_id] + run * chunk_bytes_)
          break;
        b = std::max(b, chunk_d2h_batch_[nx.chunk_id]);
        ++run;
      }
      if (b > d2h_done_upto_ && b > waited) {
        CK(cudaStreamWaitEvent(h2d_, ev_d2h_[b % kRing], 0));
        waited = b;
      }
      CK(cudaMemcpyAsync(static_cast<char*>(staging_[sb].p) + size_t(j) * chunk_bytes_, chunk_ptr_[m.chunk_id],
                         size_t(run) * chunk_bytes_, cudaMemcpyHostToDevice, h2d_));
      j += run;
    }
    CK(cudaEventRecord(ev_onload_[k], h2d_));
    if (calibrate_) CK(cudaEventRecord(ev_h2d1_[k], h2d_));
    h2d_bytes_ += uint64_t(n_on) * chunk_bytes_;
    onload_chunks_ += n_on;
  }

  // ---- compute stream ----
  CK(cudaEventRecord(ev_start_[k], comp_));
  CK(cudaStreamWaitEvent(comp_, ev_meta_[k], 0));
  const ReqDev* d_req = reinterpret_cast<const ReqDev*>(db);
  const uint32_t* d_pages = reinterpret_cast<const uint32_t*>(db + o_pages);
  const uint32_t* d_tok = reinterpret_cast<const uint32_t*>(db + o_tok);
  const uint64_t* d_kv = reinterpret_cast<const uint64_t*>(db + o_kv);
  const uint32_t* d_rr = reinterpret_cast<const uint32_t*>(db + o_rr);
  const uint32_t* d_last = reinterpret_cast<const uint32_t*>(db + o_last);
  const AttnSeg* d_segs = reinterpret_cast<const AttnSeg*>(db + o_segs);
  const AttnItem* d_items = reinterpret_cast<const AttnItem*>(db + o_items);
  const AttnPiece* d_pieces = reinterpret_cast<const AttnPiece*>(db + o_pieces);
  const uint32_t* d_ctaoff = reinterpret_cast<const uint32_t*>(db + o_ctaoff);
  const ChunkWork* d_chunks = reinterpret_cast<const ChunkWork*>(db + o_chunks);
  const uint32_t* d_creq = reinterpret_cast<const uint32_t*>(db + o_cand);
  const uint32_t* d_cid = d_creq + ncand_total;
  __nv_bfloat16* pool = static_cast<__nv_bfloat16*>(pool_.p);

  const bool prof_copy = opt_.profile != 0;
  if (prof_copy && !ev_copy_[0])
    for (auto& e : ev_copy_) CK(cudaEventCreate(&e));
  prof_scatter_ = prof_gather_ = 0;
  if (n_on) {
    CK(cudaStreamWaitEvent(comp_, ev_onload_[k], 0));
    if (prof_copy) CK(cudaEventRecord(ev_copy_[0], comp_));
    launch_scatter_chunks(pool, static_cast<const __nv_bfloat16*>(staging_[sb].p), d_chunks, d_pages, n_on, g_, comp_);
    if (prof_copy) CK(cudaEventRecord(ev_copy_[1], comp_));
    prof_scatter_ = n_on;
    ++launches;
  }
  CK(cudaEventRecord(ev_scatter_[k], comp_));

  attn_launches_last_ = 0;
  if (value_) {
    const size_t rb = size_t(rows) * d * sizeof(__nv_bfloat16);
    // comp-only workspaces: stream-ordered growth (no device synchronisation)
    if (x_.ensure(rb, comp_) || x2_.ensure(rb, comp_) || u_.ensure(rb, comp_) || q_.ensure(rb, comp_) ||
        mid_.ensure(rb, comp_) ||
        part_o_.ensure(size_t(std::max(plan_.n_slots, reduce_last ? plan_last_.n_slots : 0u)) * part_slot_floats(bq, g_.D) *
                           sizeof(float), comp_) ||
        part_lse_.ensure(size_t(std::max(plan_.n_slots, reduce_last ? plan_last_.n_slots : 0u)) * bq * sizeof(float), comp_) ||
        logits_.ensure(size_t(nr) * V * sizeof(float), comp_) ||
        scores_.ensure(size_t(ncand_total) * sizeof(float), comp_)) {
      err = "engine: workspace alloc";
      return MTKV_ERROR;
    }
    auto* X = static_cast<__nv_bfloat16*>(x_.p);
    auto* X2 = static_cast<__nv_bfloat16*>(x2_.p);
    auto* U = static_cast<__nv_bfloat16*>(u_.p);
    auto* Q = static_cast<__nv_bfloat16*>(q_.p);
    auto* MID = static_cast<__nv_bfloat16*>(mid_.p);
    if (calibrate_) {
      CK(cudaEventRecord(ev_stk0_[k], comp_));
      cal_rows_[k] = rows;
    }
    launch_embed(X, w_embed_, d_tok, rows, d, comp_);
    ++launches;
    const bool prof = opt_.profile != 0;
    if (prof && ev_attn_.size() < 4 * g_.L) {
      while (ev_attn_.size() < 4 * g_.L) {  // [0, 2L): attention pairs; [2L, 4L): projection GEMM pairs
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        ev_attn_.push_back(e);
      }
    }
    for (uint32_t l = 0; l < g_.L; ++l) {
      GemmArgs ga{};
      ga.A = X; ga.B = w_in_ + size_t(l) * d * 4 * d; ga.M = rows; ga.N = 4 * d; ga.K = d;
      ga.epi = Epi::Proj; ga.out_u = U; ga.out_q = Q; ga.pool = pool; ga.kv_off = d_kv;
      ga.layer_base = size_t(l) * g_.num_pages * 2 * S * d; ga.d = d; ga.kv_stride = S * d;
      // PDL: the prologue overlaps the previous layer's MLP; the epilogue's writes
      // (U, Q, this layer's pool plane) follow griddepcontrol.wait, by which time
      // every earlier reader of U / Q / part_o has completed (each PDL kernel of
      // the chain waited for its predecessor)
      ga.pdl = true;
      if (prof) CK(cudaEventRecord(ev_attn_[2 * g_.L + 2 * l], comp_));
      if (gemm(ga, x_.bytes / (size_t(d) * 2), err)) return MTKV_ERROR;
      if (prof) CK(cudaEventRecord(ev_attn_[2 * g_.L + 2 * l + 1], comp_));
      // the last layer (reduce_last): one query row per request, compact rows after it
      const bool last = reduce_last && l + 1 == g_.L;
      const uint32_t lrows = last ? n : rows;
      const AttnSeg* segs_l = last ? reinterpret_cast<const AttnSeg*>(db + o_segs_l) : d_segs;
      AttnArgs aa{};
      aa.q = Q; aa.pool = pool; aa.pages = d_pages; aa.segs = segs_l; aa.items = d_items;
      aa.reqs = last ? reinterpret_cast<const ReqDev*>(db + o_req_l) : d_req;
      aa.n_items = last ? n_items_l : n_items;
      aa.pieces = last ? reinterpret_cast<const AttnPiece*>(db + o_pieces_l) : d_pieces;
      aa.cta_off = last ? reinterpret_cast<const uint32_t*>(db + o_ctaoff_l) : d_ctaoff;
      aa.part_o = static_cast<float*>(part_o_.p); aa.part_lse = static_cast<float*>(part_lse_.p);
      aa.pair = last ? 0u : uint32_t(plan_.pair);
      aa.g = g_; aa.layer = l; aa.bq = bq; aa.scale_log2 = float(1.4426950408889634 / std::sqrt(double(g_.D)));
      if (prof) CK(cudaEventRecord(ev_attn_[2 * l], comp_));
      if (tc && trace_path_ && l == 0) {  // MTKV_ATTN_TRACE: per-CTA timelines of layer 0
        if (!trace_.p && trace_.ensure(size_t(kTraceCtas) * kTraceKinds * kTraceTiles * 8)) {
          err = "engine: trace alloc";
          return MTKV_ERROR;
        }
        CK(cudaMemsetAsync(trace_.p, 0, trace_.bytes, comp_));
        aa.trace = static_cast<unsigned long long*>(trace_.p);
      }
      if (tc) {
        if (pool_map_ptr_ != pool_.p || pool_map_pages_ != g_.num_pages) {
          if (make_pool_map(&pool_map_, pool_.p, g_)) { err = "engine: cuTensorMapEncodeTiled failed"; return MTKV_ERROR; }
          pool_map_ptr_ = pool_.p;
          pool_map_pages_ = g_.num_pages;
        }
        if (q_map_ptr_ != q_.p || q_map_bytes_ != q_.bytes) {
          if (make_q_map(&q_map_, q_.p, q_.bytes / (size_t(d) * sizeof(__nv_bfloat16)), g_)) {
            err = "engine: cuTensorMapEncodeTiled (queries) failed";
            return MTKV_ERROR;
          }
          q_map_ptr_ = q_.p;
          q_map_bytes_ = q_.bytes;
        }
      }
      launch_attention_any(attn_kind_, pool_map_, q_map_, aa, comp_);
      if (prof) CK(cudaEventRecord(ev_attn_[2 * l + 1], comp_));
      ++attn_launches_last_;
      GateArgs gn{};
      gn.part_o = aa.part_o; gn.part_lse = aa.part_lse; gn.segs = segs_l; gn.bm = bq; gn.u = U; gn.ln_scale = w_ln_ + size_t(l) * d;
      gn.out = X2; gn.rows = lrows; gn.H = H; gn.D = g_.D;
      if (last) {  // compact row r <- request r's last row (row-per-warp kernel)
        const uint32_t* rowc = reinterpret_cast<const uint32_t*>(db + o_rowc);
        gn.reqs = reinterpret_cast<const ReqDev*>(db + o_req_g);
        gn.row_req = rowc;
        gn.u_rows = rowc + n;
      } else {
        gn.reqs = d_req;
        gn.row_req = d_rr;
        gn.blocks = reinterpret_cast<const uint32_t*>(db + o_gblk);
        gn.n_blocks = n_gblk;
      }
      launch_gate_norm(gn, comp_);
      GemmArgs m1{};
      m1.A = X2; m1.B = w1_ + size_t(l) * d * d; m1.M = lrows; m1.N = d; m1.K = d; m1.epi = Epi::SiluBf16; m1.out = MID; m1.pdl = true;
      if (gemm(m1, x2_.bytes / (size_t(d) * 2), err)) return MTKV_ERROR;
      GemmArgs m2{};
      m2.A = MID; m2.B = w2_ + size_t(l) * d * d; m2.M = lrows; m2.N = d; m2.K = d; m2.epi = Epi::Bf16; m2.out = X; m2.pdl = true;
      if (gemm(m2, mid_.bytes / (size_t(d) * 2), err)) return MTKV_ERROR;
      launches += 5;
    }
    // the final hidden row of request r: X[last_row[r]], or X[r] after a compact last layer
    const uint32_t* lastrow = reduce_last ? reinterpret_cast<const uint32_t*>(db + o_rowc) : d_last;
    if (opt_.keep_logits || !w_out_t_) {
      // full-vocabulary logits (kept for the caller), candidates picked from them
      GemmArgs hd{};
      hd.A = X; hd.row_idx = lastrow; hd.B = w_out_; hd.M = reduce_last ? n : nr; hd.N = V; hd.K = d; hd.epi = Epi::F32;
      hd.out = logits_.p;
      launch_gemm(hd, comp_);
      ++launches;
      if (ncand_total) {
        pick_scores_kernel<<<(ncand_total + 127) / 128, 128, 0, comp_>>>(
            static_cast<float*>(scores_.p), static_cast<const float*>(logits_.p), d_creq, d_cid, ncand_total, V);
        ++launches;
      }
    } else if (ncand_total) {
      // serving: only the candidates' scores are ever read
      candidate_scores_kernel<<<(ncand_total + 7) / 8, 256, 0, comp_>>>(static_cast<float*>(scores_.p), X, w_out_t_,
                                                                      lastrow, d_creq, d_cid, ncand_total, d);
      ++launches;
    }
    if (calibrate_) CK(cudaEventRecord(ev_stk1_[k], comp_));
  } else {
    launch_tag_append(pool, d_req, d_pages, nr, max_hist, g_, comp_);
    ++launches;
  }

  // ---- offload: gather on comp (pages only ever touched here), D2H on d2h ----
  if (n_off) {
    int64_t waited = -1;
    for (uint32_t j = 0; j < n_off; ++j) {
      const int64_t b = off_slot_batch_[off_slots[j]];
      if (b > d2h_done_upto_ && b > waited) {
        CK(cudaStreamWaitEvent(comp_, ev_d2h_[b % kRing], 0));
        waited = b;
      }
    }
    if (prof_copy) CK(cudaEventRecord(ev_copy_[2], comp_));
    launch_gather_chunks(static_cast<__nv_bfloat16*>(offload_.p), pool, d_chunks + n_on, d_pages, n_off, g_, comp_);
    if (prof_copy) CK(cudaEventRecord(ev_copy_[3], comp_));
    prof_gather_ = n_off;
    ++launches;
  }
  // ---- results to the host: after the gather (kernel follows kernel on comp) and
  // ahead of the offload D2H on the copy engine (the read-back is not queued
  // behind this batch's offload burst) ----
  if (value_) {
    if (ncand_total) {
      if (scores_host_bytes_[k] < ncand_total * sizeof(float)) {
        if (scores_host_[k]) cudaFreeHost(scores_host_[k]);
        scores_host_bytes_[k] = std::max<size_t>(ncand_total * sizeof(float), 4096);
        CK(cudaHostAlloc((void**)&scores_host_[k], scores_host_bytes_[k], cudaHostAllocDefault));
      }
      CK(cudaMemcpyAsync(scores_host_[k], scores_.p, ncand_total * sizeof(float), cudaMemcpyDeviceToHost, comp_));
      d2h_bytes_ += ncand_total * sizeof(float);
    }
    if (opt_.keep_logits) {
      const size_t lb = size_t(n) * V * sizeof(float);
      if (logits_host_bytes_[k] < lb) {
        if (logits_host_[k]) cudaFreeHost(logits_host_[k]);
        logits_host_bytes_[k] = lb;
        CK(cudaHostAlloc((void**)&logits_host_[k], lb, cudaHostAllocDefault));
      }
      CK(cudaMemcpyAsync(logits_host_[k], logits_.p, lb, cudaMemcpyDeviceToHost, comp_));
      d2h_bytes_ += lb;
    }
  }
  if (n_off) {
    CK(cudaEventRecord(ev_gathered_[k], comp_));
    CK(cudaStreamWaitEvent(d2h_, ev_gathered_[k], 0));
    for (uint32_t j = 0; j < n_off; ++j) {
      const ChunkMove& m = w.offloads[j];
      if (host_chunk(m.chunk_id, m.user, m.chunk_index, err)) return MTKV_ERROR;
      CK(cudaMemcpyAsync(chunk_ptr_[m.chunk_id], static_cast<char*>(offload_.p) + size_t(off_slots[j]) * chunk_bytes_,
                         chunk_bytes_, cudaMemcpyDeviceToHost, d2h_));
      chunk_d2h_batch_[m.chunk_id] = int64_t(batch_no_);
      chunk_off_slot_[m.chunk_id] = off_slots[j];
      off_slot_batch_[off_slots[j]] = int64_t(batch_no_);
    }
    CK(cudaEventRecord(ev_d2h_[k], d2h_));
    d2h_rec_batch_[k] = int64_t(batch_no_);
    d2h_bytes_ += uint64_t(n_off) * chunk_bytes_;
    offload_chunks_ += n_off;
  }
  CK(cudaEventRecord(ev_done_[k], comp_));
  CK(cudaGetLastError());
  last_slot_ = k;
  last_n_ = n;
  ++batch_no_;
  return MTKV_OK;
}

int Engine::drain(std::string& err) {
  std::vector<uint64_t> persisted;
  planner.drain(&persisted);
  for (uint64_t id : persisted)
    if (id < chunk_off_slot_.size() && chunk_off_slot_[id] >= 0) {
      off_free_.push_back(uint32_t(chunk_off_slot_[id]));
      chunk_off_slot_[id] = -1;
    }
  (void)err;
  return MTKV_OK;
}

int Engine::synchronize(std::string& err) {
  CK(cudaSetDevice(opt_.device));
  CK(cudaStreamSynchronize(comp_));
  CK(cudaStreamSynchronize(h2d_));
  CK(cudaStreamSynchronize(d2h_));
  return MTKV_OK;
}

int Engine::last_logits(float* out, uint32_t cap_rows, std::string& err) {
  if (!value_) { err = "logits: tag backend has no model"; return MTKV_ERROR; }
  if (!opt_.keep_logits) { err = "logits: engine created without keep_logits"; return MTKV_ERROR; }
  if (last_slot_ < 0) return 0;
  CK(cudaEventSynchronize(ev_done_[last_slot_]));
  const uint32_t rows = std::min(cap_rows, last_n_);
  std::memcpy(out, logits_host_[last_slot_], size_t(rows) * opt_.model.vocab * sizeof(float));
  return int(last_n_);
}

int Engine::last_rankings(uint32_t* out, uint64_t cap, std::string& err) {
  if (last_slot_ < 0) return 0;
  return batch_rankings(batch_no_ - 1, out, cap, err);
}

int Engine::batch_rankings(uint64_t ticket, uint32_t* out, uint64_t cap, std::string& err) {
  if (!value_) { err = "rankings: tag backend has no model"; return MTKV_ERROR; }
  const int k = int(ticket % kRing);
  if (ticket >= batch_no_ || slot_batch_[k] != int64_t(ticket)) {
    err = "rankings: results of batch " + std::to_string(ticket) + " are not available (only the last " +
          std::to_string(kRing) + " submitted batches are kept)";
    return MTKV_ERROR;
  }
  CK(cudaEventSynchronize(ev_done_[k]));
  const float* sc = scores_host_[k];
  const std::vector<uint32_t>& cands = slot_cands_[k];
  const std::vector<uint32_t>& nc = slot_nc_[k];
  uint64_t o = 0;
  size_t base = 0;
  std::vector<uint32_t> idx;
  for (uint32_t r = 0; r < nc.size(); ++r) {
    idx.resize(nc[r]);
    for (uint32_t i = 0; i < nc[r]; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) { return sc[base + a] > sc[base + b]; });
    for (uint32_t i : idx)
      if (o < cap) out[o++] = cands[base + i];
    base += nc[r];
  }
  return int(o);
}

int64_t Engine::read_user_kv(uint32_t user, uint32_t layer, uint16_t* kout, uint16_t* vout, uint64_t cap,
                             std::string& err) {
  if (synchronize(err)) return -1;
  const UserRec* u = planner.find(user);
  if (!u || !u->known) { err = "read_user_kv: unknown user"; return -1; }
  if (layer >= g_.L) { err = "read_user_kv: bad layer"; return -1; }
  const uint64_t n = std::min<uint64_t>(u->device_len, cap);
  const size_t seg = size_t(g_.S) * g_.d;
  std::vector<uint16_t> buf(2 * seg);
  for (uint64_t pos = 0; pos < n; pos += g_.S) {
    const uint32_t page = u->pages[pos / g_.S];
    const size_t o = g_.off(layer, page, 0, 0);
    if (cudaMemcpy(buf.data(), static_cast<__nv_bfloat16*>(pool_.p) + o, 2 * seg * 2, cudaMemcpyDeviceToHost) != cudaSuccess) {
      err = "read_user_kv: copy failed";
      return -1;
    }
    const uint64_t take = std::min<uint64_t>(g_.S, n - pos);
    std::memcpy(kout + pos * g_.d, buf.data(), take * g_.d * 2);
    std::memcpy(vout + pos * g_.d, buf.data() + seg, take * g_.d * 2);
  }
  return int64_t(n);
}

int Engine::check_conservation(std::string& err) {
  if (value_) { err = "conservation check uses the tag backend"; return MTKV_ERROR; }
  if (synchronize(err)) return MTKV_ERROR;
  const uint32_t L = g_.L, d = g_.d, C = g_.chunk;
  for (uint32_t uid : planner.known_users()) {
    const UserRec* u = planner.find(uid);
    if (u->persisted_len % C) { err = "conservation: persisted length not chunk-aligned"; return MTKV_ERROR; }
    if (u->pages.size() * uint64_t(g_.S) < u->device_len) { err = "conservation: device length exceeds page table"; return MTKV_ERROR; }
    std::vector<uint16_t> kb(u->device_len * d + 1), vb(u->device_len * d + 1);
    for (uint32_t l = 0; l < L; ++l) {
      if (read_user_kv(uid, l, kb.data(), vb.data(), u->device_len, err) < 0) return MTKV_ERROR;
      for (uint64_t pos = 0; pos < u->device_len; ++pos)
        for (uint32_t j = 0; j < d; ++j)
          if (kb[pos * d + j] != tag_word(uid, pos, l, 0, j) || vb[pos * d + j] != tag_word(uid, pos, l, 1, j)) {
            err = "conservation: wrong identity on device (user " + std::to_string(uid) + ", pos " +
                  std::to_string(pos) + ", layer " + std::to_string(l) + ")";
            return MTKV_ERROR;
          }
    }
    if (u->host_chunks.size() != u->persisted_len / C) { err = "conservation: host chunk count disagrees"; return MTKV_ERROR; }
    for (size_t c = 0; c < u->host_chunks.size(); ++c) {
      const uint16_t* hc = reinterpret_cast<const uint16_t*>(chunk_ptr_[u->host_chunks[c]]);
      for (uint32_t l = 0; l < L; ++l)
        for (uint32_t kv = 0; kv < 2; ++kv)
          for (uint32_t t = 0; t < C; ++t)
            for (uint32_t j = 0; j < d; ++j)
              if (hc[((size_t(l) * 2 + kv) * C + t) * d + j] != tag_word(uid, c * C + t, l, kv, j)) {
                err = "conservation: wrong identity on host (user " + std::to_string(uid) + ")";
                return MTKV_ERROR;
              }
    }
  }
  return MTKV_OK;
}

double Engine::last_batch_ms() {
  if (last_slot_ < 0) return 0;
  cudaEventSynchronize(ev_done_[last_slot_]);
  float ms = 0;
  cudaEventElapsedTime(&ms, ev_start_[last_slot_], ev_done_[last_slot_]);
  return ms;
}

double Engine::last_attention_ms(uint32_t* n) {
  if (n) *n = attn_launches_last_;
  if (trace_path_ && trace_.p && last_slot_ >= 0) {
    cudaEventSynchronize(ev_done_[last_slot_]);
    std::vector<unsigned long long> h(trace_.bytes / 8);
    cudaMemcpy(h.data(), trace_.p, trace_.bytes, cudaMemcpyDeviceToHost);
    if (FILE* f = std::fopen(trace_path_, "wb")) {
      std::fwrite(h.data(), 8, h.size(), f);
      std::fclose(f);
    }
  }
  if (last_slot_ < 0 || !opt_.profile || ev_attn_.empty()) return 0;
  cudaEventSynchronize(ev_done_[last_slot_]);
  double tot = 0;
  for (uint32_t l = 0; l < attn_launches_last_ && 2 * l + 1 < ev_attn_.size(); ++l) {
    float ms = 0;
    cudaEventElapsedTime(&ms, ev_attn_[2 * l], ev_attn_[2 * l + 1]);
    tot += ms;
  }
  return tot;
}

double Engine::last_proj_ms(uint32_t* launches, uint64_t* rows) {
  *launches = 0;
  *rows = last_rows_;
  if (last_slot_ < 0 || !opt_.profile || ev_attn_.size() < 4 * g_.L || !value_) return 0;
  cudaEventSynchronize(ev_done_[last_slot_]);
  double tot = 0;
  for (uint32_t l = 0; l < g_.L; ++l) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, ev_attn_[2 * g_.L + 2 * l], ev_attn_[2 * g_.L + 2 * l + 1]) == cudaSuccess) {
      tot += ms;
      ++*launches;
    }
  }
  return tot;
}

int Engine::last_chunk_copy_ms(double* scatter_ms, uint32_t* scatter_chunks, double* gather_ms,
                               uint32_t* gather_chunks) {
  *scatter_ms = *gather_ms = 0;
  *scatter_chunks = *gather_chunks = 0;
  if (last_slot_ < 0 || !opt_.profile || !ev_copy_[0]) return MTKV_OK;
  cudaEventSynchronize(ev_done_[last_slot_]);
  float ms = 0;
  if (prof_scatter_ && cudaEventElapsedTime(&ms, ev_copy_[0], ev_copy_[1]) == cudaSuccess) {
    *scatter_ms = ms;
    *scatter_chunks = prof_scatter_;
  }
  if (prof_gather_ && cudaEventElapsedTime(&ms, ev_copy_[2], ev_copy_[3]) == cudaSuccess) {
    *gather_ms = ms;
    *gather_chunks = prof_gather_;
  }
  return MTKV_OK;
}

void Engine::report(mtkv_run_report& r) const {
  planner.report(r);
  r.h2d_bytes = h2d_bytes_;
  r.d2h_bytes = d2h_bytes_;
  r.onload_chunks = onload_chunks_;
  r.offload_chunks = offload_chunks_;
}

}  // namespace mtkv_b200
