// GPU engine = Planner (host control plane) + executor (B200 data plane).
//
// Streams (paper §4.4 four lanes, mapped onto B200 engines):
//   comp : scatter, per-layer GEMM/append/attention/norm, logits, offload gathers
//   h2d  : copy-engine onload of host chunks into a staging slot ring
//   d2h  : copy-engine offload of gathered chunks into the pinned host store
// The planner never waits for the device, so the onload copies of batch i+1
// are enqueued while batch i still computes (cross-batch overlap); the only
// cross-stream edges are the three hazards documented in engine.cu.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "kernels.cuh"
#include "planner.hpp"

namespace mtkv_b200 {

constexpr int kRing = 6;  // batches in flight on the device (and results kept for rankings)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool async = false;        // allocated stream-ordered
  // grows when needed: stream-ordered on `s` when the buffer is only used on
  // that stream, else device-synchronising
  int ensure(size_t need, cudaStream_t s = nullptr);
  void release();
};

class Engine {
 public:
  Engine(const mtkv_kv_config& kv, const mtkv_cost_model& cost, const mtkv_engine_options& opt);
  ~Engine();
  int init(std::string& err);

  int process_batch(const mtkv_request* reqs, uint32_t n, std::string& err);
  int drain(std::string& err);
  int synchronize(std::string& err);
  int last_logits(float* out, uint32_t cap_rows, std::string& err);
  int last_rankings(uint32_t* out, uint64_t cap, std::string& err);
  // rankings of an earlier batch (ticket = 0-based submission index) while later
  // batches are in flight; valid for the last kRing submitted batches
  int batch_rankings(uint64_t ticket, uint32_t* out, uint64_t cap, std::string& err);
  uint64_t batches_submitted() const { return batch_no_; }
  // wall time of the last batch's control plane (host planner, including the
  // device planner's round trip when enabled) and the device planner kernel time
  void last_plan_ms(double* plan_ms, double* ctl_kernel_ms) const {
    *plan_ms = last_plan_ms_;
    *ctl_kernel_ms = planner.device_ctl() ? ctl_.last_kernel_ms() : 0.0;
  }
  int check_conservation(std::string& err);
  int64_t read_user_kv(uint32_t user, uint32_t layer, uint16_t* k, uint16_t* v, uint64_t cap,
                       std::string& err);
  double last_batch_ms();
  double last_attention_ms(uint32_t* launches);
  int gemm(const GemmArgs& a, uint64_t a_rows_alloc, std::string& err);
  // profile mode: device time of the last batch's onload scatter and offload gather
  int last_chunk_copy_ms(double* scatter_ms, uint32_t* scatter_chunks, double* gather_ms, uint32_t* gather_chunks);
  // profile mode: device ms of the last batch's projection GEMMs (with the fused paged K/V append)
  double last_proj_ms(uint32_t* launches, uint64_t* rows);
  void report(mtkv_run_report& r) const;
  void set_profile(uint32_t on) { opt_.profile = on; }
  int set_onload_policy(uint32_t policy, double gbs, double mtok_s, std::string& err);
  uint32_t batch_size() const { return opt_.batch_size ? opt_.batch_size : 1; }

  Planner planner;
  uint64_t launches = 0;

 private:
  int enqueue(const BatchWork& w, const mtkv_request* reqs, uint32_t n, std::string& err);
  int validate_payload(const mtkv_request* reqs, uint32_t n, std::string& err) const;
  int host_chunk(uint64_t id, uint32_t user, uint32_t index, std::string& err);  // pinned storage
  char* take_slab();
  void slab_refill_loop();
  void init_weights();

  mtkv_kv_config kv_;
  mtkv_engine_options opt_;
  PoolGeom g_{};
  size_t chunk_elems_ = 0, chunk_bytes_ = 0;
  bool value_ = false, recompute_ = false;

  cudaStream_t comp_ = nullptr, h2d_ = nullptr, d2h_ = nullptr;
  cudaEvent_t ev_onload_[kRing], ev_scatter_[kRing], ev_gathered_[kRing], ev_d2h_[kRing],
      ev_done_[kRing], ev_start_[kRing], ev_meta_[kRing];
  // adaptive-policy calibration: per ring slot, the layer stack's span on comp
  // (embed -> scores) and the onload copies' span on h2d, with the rows / bytes
  // they processed; read back when the slot is reused (the batch is complete)
  cudaEvent_t ev_stk0_[kRing], ev_stk1_[kRing], ev_h2d0_[kRing], ev_h2d1_[kRing];
  uint64_t cal_rows_[kRing] = {}, cal_bytes_[kRing] = {};
  double cal_tps_ = 0, cal_Bps_ = 0;  // EMAs (0: no measurement yet)
  bool calibrate_ = false;            // adaptive policy with no fixed rates given
  void calibrate_from(int k);
  std::vector<cudaEvent_t> ev_attn_;  // profiling pairs of the last batch
  cudaEvent_t ev_copy_[4] = {nullptr, nullptr, nullptr, nullptr};  // scatter start/end, gather start/end
  uint32_t prof_scatter_ = 0, prof_gather_ = 0;
  uint32_t attn_launches_last_ = 0;
  uint64_t batch_no_ = 0;
  int64_t last_slot_ = -1;
  bool have_scatter_[kRing] = {};
  bool have_d2h_[kRing] = {};
  int64_t scatter_batch_[kRing];  // -1: none (constructor)

  // device memory
  DevBuf pool_, staging_[2], offload_, meta_, x_, x2_, u_, q_, mid_, part_o_, part_lse_, logits_, scores_;
  __nv_bfloat16 *w_embed_ = nullptr, *w_in_ = nullptr, *w1_ = nullptr, *w2_ = nullptr, *w_out_ = nullptr;
  __nv_bfloat16* w_out_t_ = nullptr;  // w_out transposed [V x d] (candidate scores)
  float* w_ln_ = nullptr;
  uint32_t staging_slots_ = 0;
  bool use_tc_ = false;          // a tcgen05 attention kernel (attn_kind_ != Mma)
  AttnKind attn_kind_ = AttnKind::Mma;
  int n_sm_ = 1;                 // persistent attention CTAs
  DevCtl ctl_;                   // device control plane (opt_.device_planner)
  double last_plan_ms_ = 0;
  uint64_t last_rows_ = 0;
  AttnPlan plan_;                // attention plan of the batch being enqueued
  AttnPlan plan_last_;           // ... of its last layer (one query row per request)
  const char* trace_path_ = std::getenv("MTKV_ATTN_TRACE");
  DevBuf trace_;
  alignas(64) CUtensorMap pool_map_{};
  alignas(64) CUtensorMap q_map_{};
  const void* pool_map_ptr_ = nullptr;
  uint32_t pool_map_pages_ = 0;
  const void* q_map_ptr_ = nullptr;
  size_t q_map_bytes_ = 0;

  // pinned host memory: slabs -> per-user extents -> chunks
  static constexpr size_t kSpareSlabs = 2;
  std::vector<char*> slabs_, spare_slabs_;
  std::mutex slab_mu_;
  std::condition_variable slab_cv_;
  std::thread refill_;
  bool stop_refill_ = false;
  char* cur_slab_ = nullptr;
  size_t slab_bytes_ = 0, slab_used_ = 0;
  uint32_t chunks_per_extent_ = 1;
  std::unordered_map<uint32_t, std::vector<char*>> user_extents_;
  std::vector<char*> chunk_ptr_;          // chunk id -> pinned [L][2][chunk][d]
  std::vector<int64_t> chunk_d2h_batch_;  // batch whose d2h ring event covers the chunk
  std::vector<uint32_t> off_free_;        // free offload slots
  std::vector<int64_t> off_slot_batch_;   // last batch that used each offload slot
  std::vector<int64_t> chunk_off_slot_;   // chunk id -> offload slot while in flight
  // ev_d2h_ slots are reused every kRing batches: a batch that left the ring has
  // its D2H confirmed on the host (d2h_done_upto_), so waits only ever target
  // batches still in the ring and never alias a newer record of the same slot
  int64_t d2h_rec_batch_[kRing];  // batch that last recorded ev_d2h_[k] (-1: none; constructor)
  int64_t d2h_done_upto_ = -1;
  char* meta_host_[kRing] = {};
  size_t meta_host_bytes_[kRing] = {};
  size_t meta_slot_ = 0;  // bytes per ring slot of the device metadata buffer (256-B multiple)
  float* scores_host_[kRing] = {};
  size_t scores_host_bytes_[kRing] = {};
  float* logits_host_[kRing] = {};
  size_t logits_host_bytes_[kRing] = {};

  // last batch bookkeeping for logits / rankings
  uint32_t last_n_ = 0;
  // per ring slot: candidate ids and counts of the batch whose scores it holds
  std::vector<uint32_t> slot_cands_[kRing], slot_nc_[kRing];
  int64_t slot_batch_[kRing];  // -1: none (constructor)
  uint64_t h2d_bytes_ = 0, d2h_bytes_ = 0, onload_chunks_ = 0, offload_chunks_ = 0;
};

}  // namespace mtkv_b200
