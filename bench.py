"""Serving-path benchmark (BASELINE.json metric) — one JSON line on rank 0.

Workload (BASELINE.json configs[1]): GR model 4 layers, d=256 (H=2, D=128),
users with 4K-token histories, 64 new tokens + 8 candidates per request,
device page pool sized to ~10% of the user population's KV, pinned-host
backup tier (chunked store), hierarchical mode. A "step" is one batch of
requests through the full hot path: plan (LRU/eviction/allocation), H2D
onload of host hits, scatter, per-layer fused projection + paged KV append,
incremental prefix-reuse attention, norm/MLP, scoring head, offload of full
chunks (gather + D2H).

Warm-up (untimed): prefill of every user's 4K history through the same
engine, then W revisit batches. Timed: K revisit batches. Synthetic data
(random token ids, reference-initialised random weights).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1: launched by torchrun, one process per GPU; users are sharded by
user-id hash (paper_2604_22881_b200.shard.shard_of), each rank owns an
independent cache shard; no collective on the data path ("scaling": "weak").

Host hits are executed with the `adaptive` policy by default (`--onload-policy
always` is the reference's executor): every host hit re-encodes its earliest
chunks on the SMs and onloads the rest, balanced at measured rates; the
control plane, hit ratios and simulated clock are the reference's under both
("Host-hit executor policy"); phase E reports the other policy.

Phases: A = device throughput (`value`, pre-packed requests, CUDA events);
B = per-batch latency (p50/p99, `always` policy) with per-kernel CUDA-event
timing of the attention launches (`roofline`: the decode-shaped incremental
attention), the projection GEMM and the KV scatter/gather (`other_kernels`);
C = end to end through the public API (`e2e`: Python request dicts -> C-ABI,
pipelined submit / rankings read-back of every batch, 3 batches in flight);
D (untimed) = 8 more batches under CUPTI for `overlap` (fraction of kernel
time with an H2D copy in flight, H2D engine busy fraction) and the copy
kernels' own durations; E = the other host-hit policy on the next K batches.
Also reported: `host_link` (H2D GB/s vs the measured pinned-copy peak),
`control_plane` (planning cost; `--planner device` runs the GPU control
plane), `cpu_baseline` (the unmodified reference on this box's host cores).
Other BASELINE configs: `--config gr8_d512` (configs[3] per-GPU shard),
`--config tiny_d64` (configs[0]), `--mode recompute|gpu_only` (configs[2]),
`--pool-frac F` (configs[4]); tools/configs_sweep.sh runs them.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "requests/sec & tokens/sec at fixed hit ratio, p99 latency, 1/2/4/8 B200 vs CPU"
# MTKV_BENCH_ONE_GPU=1: all torchrun ranks on GPU 0 (functional check of the sharded
# multi-rank flow on a one-GPU box; its throughput is not a scaling number)
ONE_GPU = os.environ.get("MTKV_BENCH_ONE_GPU") == "1"
H2D_PEAK_GBS = 55.5  # measured pinned H2D, 64-256 MiB copies (profiles/r01_probe_h2d.json)

CONFIGS = {
    # BASELINE.json configs[1] — the headline single-GPU workload
    "gr4_d256": dict(L=4, H=2, D=128, vocab=4096, users=2048, history=4096, delta=64, cands=8,
                     page=32, chunk=128, pool_frac=0.10, batch=64),
    # configs[0] — the reference's smallest CPU case (parity-test sized)
    "tiny_d64": dict(L=2, H=2, D=32, vocab=512, users=256, history=1024, delta=32, cands=8,
                     page=32, chunk=128, pool_frac=0.10, batch=32),
    # configs[3] per GPU shard — production-scale model (8-layer d=512, 8K histories);
    # 256 users per GPU keep the pinned host tier at ~35 GB per process
    "gr8_d512": dict(L=8, H=4, D=128, vocab=4096, users=256, history=8192, delta=64, cands=8,
                     page=32, chunk=128, pool_frac=0.10, batch=16),
}


def LAST_LAYER_REDUCED(cfg) -> bool:
    """The engine's tcgen05 attention path (head_dim 64/128, not forced to another
    kernel by MTKV_ATTN) runs the last layer for each request's last row only."""
    return (cfg["D"] in (64, 128) and os.environ.get("MTKV_ATTN", "") not in ("mma", "pp")
            and not os.environ.get("MTKV_LAST_LAYER", "").startswith("f"))


CONFIG_TAG = {"gr4_d256": "configs[1]", "tiny_d64": "configs[0]", "gr8_d512": "configs[3]"}


def bind_host_to_gpu(local: int):
    """Multi-GPU ranks: run this rank's host threads on the CPUs NVML reports as
    close to its GPU, so the pinned host tier (first-touched by this thread and
    the slab-refill thread it starts) sits on the GPU's NUMA node and each
    GPU's PCIe link streams from local memory. Best effort: returns a short
    description, or None when NVML or the topology gives nothing to do."""
    try:
        import pynvml
        import torch
        p = torch.cuda.get_device_properties(local)
        bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        ncpu = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = {64 * w + b for w, m in enumerate(words) for b in range(64) if (int(m) >> b) & 1}
        cur = os.sched_getaffinity(0)
        near = cpus & cur
        if not near or near == cur:
            return None
        os.sched_setaffinity(0, near)
        return f"{len(near)} of {len(cur)} cpus near {bus}"
    except Exception:  # no NVML / no affinity information: leave the scheduler alone
        return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.lines = gpu, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout: float = 5.0):
        """nvidia-smi's start-up (NVML init) can hold the driver for up to ~1 s:
        let it finish before a timed region starts (sampling continues inside it)."""
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.02)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_workload(cfg: dict, n_batches: int, rank: int, world: int, seed: int = 1):
    """Prefill requests (one 4K-token first visit per user) + revisit stream.

    Revisits follow the reference generator's heavy-tailed (lognormal) return
    process (workload.cpp:85, fixed_delta=Δ): recently active users come back
    soon — the temporal locality the LRU policy exploits. The first part of the
    stream is consumed as warm-up so the timed phases see the steady state."""
    import paper_2604_22881_b200 as mtkv
    from paper_2604_22881_b200.shard import shard_of
    rng = np.random.default_rng(seed + 7919 * rank)
    U, V = cfg["users"], cfg["vocab"]
    # user-id hash sharding across ranks (paper_2604_22881_b200.shard): this
    # rank's users are the first U ids that hash to it
    ids, u = [], 0
    while len(ids) < U:
        if shard_of(u, world) == rank:
            ids.append(u)
        u += 1
    uid = lambda u: ids[u]
    prefill = [{"ts": 0, "user": uid(u), "dn": cfg["history"], "nc": cfg["cands"],
                "tokens": rng.integers(0, V, cfg["history"], dtype=np.uint32),
                "cands": rng.integers(0, V, cfg["cands"], dtype=np.uint32)} for u in range(U)]
    n_rev = n_batches * cfg["batch"]
    revisits = []
    for ts, u in stationary_revisits(U, n_rev, rng):
        revisits.append({"ts": int(ts), "user": uid(int(u)), "dn": cfg["delta"], "nc": cfg["cands"],
                         "tokens": rng.integers(0, V, cfg["delta"], dtype=np.uint32),
                         "cands": rng.integers(0, V, cfg["cands"], dtype=np.uint32)})
    return prefill, revisits


def stationary_revisits(U: int, n: int, rng, mu: float = 9.0, sigma: float = 1.6):
    """Per-user renewal processes with lognormal return gaps (ms) — the heavy
    tail of the paper's Fig. 5 and of the reference presets (workload.cpp:28,
    gap_log_mu=9, gap_log_sigma=1.6) — merged in time, observed after a burn-in
    of several mean gaps so the window is stationary (the reference generator's
    fixed horizon is not: its traffic ramps up and down)."""
    mean_gap = np.exp(mu + sigma ** 2 / 2)
    window = n * mean_gap / U * 1.05
    t0 = 6 * mean_gap
    horizon = t0 + window
    per_user = int(horizon / mean_gap * 1.6) + 32
    gaps = np.exp(rng.normal(mu, sigma, size=(U, per_user)))
    times = np.cumsum(gaps, axis=1) - rng.uniform(0, mean_gap, size=(U, 1))
    users = np.broadcast_to(np.arange(U)[:, None], times.shape)
    sel = (times >= t0) & (times < horizon)
    t, u = times[sel], users[sel]
    order = np.argsort(t, kind="stable")
    t, u = t[order][:n], u[order][:n]
    if len(t) < n:  # extremely unlikely; pad by recycling the window
        reps = -(-n // len(t))
        t = np.concatenate([t + k * window for k in range(reps)])[:n]
        u = np.tile(u, reps)[:n]
    return zip(t - t0, u)


def kv_config(cfg):
    import paper_2604_22881_b200 as mtkv
    pages_per_user = -(-(cfg["history"] + 16 * cfg["delta"]) // cfg["page"])
    # ~pool_frac of the population's KV, but never less than two batches of users
    device_pages = max(int(cfg["pool_frac"] * cfg["users"] * pages_per_user),
                       2 * cfg["batch"] * pages_per_user) + 4 * cfg["batch"]
    chunks_per_batch = cfg["batch"] * (-(-cfg["history"] // cfg["chunk"]) + 2)
    return mtkv.KVConfig(num_layers=cfg["L"], num_heads=cfg["H"], head_dim=cfg["D"], page_size=cfg["page"],
                         chunk_size=cfg["chunk"], device_pages=device_pages,
                         onload_pages=chunks_per_batch * (cfg["chunk"] // cfg["page"]),
                         offload_quota=cfg["chunk"] * 4 * chunks_per_batch)


def _phase(r0, r1, steps, B):
    req = r1["hist_required"] - r0["hist_required"]
    dev = r1["hist_device"] - r0["hist_device"]
    host = r1["hist_host"] - r0["hist_host"]
    return {"gpu_hit": dev / req if req else 1.0, "total_hit": (dev + host) / req if req else 1.0,
            "h2d_bytes_per_step": (r1["h2d_bytes"] - r0["h2d_bytes"]) / steps,
            "d2h_bytes_per_step": (r1["d2h_bytes"] - r0["d2h_bytes"]) / steps,
            "onload_chunks_per_step": (r1["onload_chunks"] - r0["onload_chunks"]) / steps,
            "fresh_tokens": r1["tokens_processed"] - r0["tokens_processed"],
            "prefix_recomputed_frac": (r1["prefix_recomputed"] - r0["prefix_recomputed"]) / max(
                1, (r1["prefix_recomputed"] - r0["prefix_recomputed"]) + (r1["prefix_onloaded"] - r0["prefix_onloaded"])),
            "evictions": r1["evictions"] - r0["evictions"]}


def run_b200(args, cfg):
    import torch
    import paper_2604_22881_b200 as mtkv
    world, rank, local = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist
        if ONE_GPU:  # functional check of the N>1 path on a one-GPU box: ranks share GPU 0, gloo reductions
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if ONE_GPU:
        local = 0
    torch.cuda.set_device(local)
    numa = bind_host_to_gpu(local) if world > 1 and not ONE_GPU else None
    # the pinned host tier holds every user's persisted prefix (~90 % of the KV
    # working set): on a box whose RAM cannot pin world x that, each rank serves
    # proportionally fewer users (recorded in the line) instead of failing
    host_note = None
    if args.mode == "hierarchical":
        per_user_mb = -(-((cfg["history"] + 16 * cfg["delta"]) * 2 * cfg["L"] * cfg["H"] * cfg["D"] * 2) // 2**20)
        try:
            ram_mb = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") // 2**20
        except (ValueError, OSError):
            ram_mb = 0
        need_mb = world * (1.1 * cfg["users"] * per_user_mb + 1024)  # every rank of this launch is on this box
        if ram_mb and need_mb > 0.75 * ram_mb:
            users = max(cfg["batch"] * 4, int(cfg["users"] * 0.75 * ram_mb / need_mb))
            host_note = f"users per rank {cfg['users']} -> {users}: {world} ranks x pinned tier exceed 75% of {ram_mb} MB RAM"
            cfg["users"] = users
    kv = kv_config(cfg)
    cost = mtkv.CostModel(bus_bandwidth=55e9)  # measured pinned H2D on the B200 box (probe)
    model = mtkv.ModelConfig(num_layers=cfg["L"], num_heads=cfg["H"], head_dim=cfg["D"], vocab=cfg["vocab"],
                             seed=1)
    B, K = cfg["batch"], args.steps
    warm = args.warmup + max(args.warmup, 2 * K)  # long warm-up: timed phases see the steady state
    N_OVL = 8  # phase D batches (compute / transfer overlap under CUPTI)
    prefill, revisits = make_workload(cfg, warm + 4 * K + N_OVL, rank, world)
    # pinned host store sized for the run up front (no cudaHostAlloc while serving)
    tok_bytes = kv.token_kv_bytes()
    # one pinned extent per user sized to its persisted prefix over the run, so a
    # user's onload is a single large copy-engine transfer (host-link peak)
    extent_mb = -(-((cfg["history"] + 16 * cfg["delta"]) * tok_bytes) // 2**20)
    host_mb = int(1.1 * cfg["users"] * extent_mb) + 1024
    ppu = -(-(cfg["history"] + 16 * cfg["delta"]) // cfg["page"])
    hier = args.mode == "hierarchical"
    eng = mtkv.Engine(kv, cost, mode=args.mode, backend="value", batch_size=B, model=model,
                      device=local, host_reserve_mb=host_mb if hier else 0, host_extent_mb=extent_mb,
                      planner=args.planner, max_users=cfg["users"] + 64, max_user_pages=2 * ppu + 64,
                      onload_policy=args.onload_policy)
    # ---- warm-up: prefill histories (untimed), then the first revisit batches ----
    pb = max(1, min(cfg["batch"], 65536 // cfg["history"]))  # prefill batches fit the pool like serving ones
    for i in range(0, len(prefill), pb):
        eng.process_batch(prefill[i:i + pb])
    batches = [revisits[i * B:(i + 1) * B] for i in range(warm + 4 * K + N_OVL)]
    packed = [mtkv.RequestBatch(b) for b in batches]
    for i in range(warm):
        eng.process_batch(None, packed=packed[i])
    eng.synchronize()
    if dist:
        dist.barrier()

    # ---- phase A (value): device throughput, requests pre-packed in host memory ----
    r0 = eng.report()
    l0 = eng.kernel_launches()
    clocks = Clocks(local)
    clocks.start()
    clocks.wait_first()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record()
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" selects these launches
    for i in range(warm, warm + K):
        eng.process_batch(None, packed=packed[i])
    eng.synchronize()
    torch.cuda.nvtx.range_pop()
    t_end.record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    r1 = eng.report()
    elapsed = t_start.elapsed_time(t_end) / 1e3
    launches_per_step = (eng.kernel_launches() - l0) / K
    phase_a = _phase(r0, r1, K, B)

    # ---- phase C (e2e): public API with Python request dicts, every step's rankings read back ----
    # (right after phase A: the adaptive policy's calibrated rates are phase A's;
    # phase B runs the `always` policy with per-launch events)
    # pipelined serving: batch i's rankings are read (D2H + host ranking) while
    # batches i+1 .. i+depth are in flight, as a server overlapping requests
    # would (the engine keeps the results of its last 6 batches; the next
    # batch's onload must be queued before the link drains: depth 3 measured
    # 17.4 K vs 12.7 K requests/s at depth 2, tools/probe_timing.py; default 5)
    e0 = eng.report()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    w0 = time.perf_counter()
    kc = warm + K
    pending, n_read, e2e_wait = [], 0, 0.0
    depth = max(1, min(5, args.e2e_depth))
    for i in range(kc, kc + K):
        pending.append(eng.submit(batches[i]))   # host dicts -> C-ABI (packing + H2D inside)
        if len(pending) > depth:
            wt = time.perf_counter()
            eng.rankings(pending.pop(0))
            e2e_wait += time.perf_counter() - wt
            n_read += 1
    for t in pending:
        eng.rankings(t)
        n_read += 1
    eng.synchronize()
    e2e_s = time.perf_counter() - w0
    if dist:
        dist.barrier()
    assert n_read == K
    phase_c = _phase(e0, eng.report(), K, B)


    # ---- phase B: per-batch device latency (p50/p99) + per-launch attention timing ----
    # (host hits onloaded: the incremental attention the roofline describes; the
    # adaptive policy's re-encoded prefixes are prefill-shaped, tensor-bound rows)
    eng.set_onload_policy("always")
    eng.set_profile(True)
    eng_lat, attn_ms, attn_launches, attn_bytes = [], 0.0, 0, 0
    copy_stat = [0.0, 0, 0.0, 0, 0, 0]  # scatter ms, chunks, gather ms, chunks, launches, launches
    plan_ms, ctl_ms = [], []
    proj_stat = [0.0, 0, 0]  # projection GEMM ms, launches, rows (summed over launches)
    d = cfg["H"] * cfg["D"]
    rb0 = eng.report()
    k0 = warm + 2 * K
    for i in range(k0, k0 + K):
        eng.process_batch(None, packed=packed[i])
        eng.synchronize()
        eng_lat.append(eng.last_batch_ms())
        ms, n = eng.last_attention_ms()
        attn_ms += ms
        attn_launches += n
        pm, km = eng.last_plan_ms()
        plan_ms.append(pm)
        ctl_ms.append(km)
        pm_, pn_, prow_ = eng.last_proj_ms()
        proj_stat[0] += pm_; proj_stat[1] += pn_; proj_stat[2] += prow_ * pn_
        sm, sc, gm, gc = eng.last_chunk_copy_ms()
        copy_stat[0] += sm; copy_stat[1] += sc; copy_stat[2] += gm; copy_stat[3] += gc
        copy_stat[4] += 1 if sc else 0; copy_stat[5] += 1 if gc else 0
        plans = eng.plans()
        # the last layer computes only each request's last row (tcgen05 path,
        # batches of >= 4096 fresh rows: engine.cu reduce_last)
        reduced = LAST_LAYER_REDUCED(cfg) and sum(
            p["fresh_history"] + p["delta"] + p["num_candidates"] for p in plans) >= 4096
        for p in plans:
            keys = p["history_len"] + p["delta"] + p["num_candidates"]
            rows = p["fresh_history"] + p["delta"] + p["num_candidates"]
            # per layer: K+V of every visible key once + Q (bf16) read + O (fp32) write
            last_rows = 1 if reduced else rows
            attn_bytes += (cfg["L"] - 1) * (keys * d * 2 * 2 + rows * d * 2 + rows * d * 4)
            attn_bytes += keys * d * 2 * 2 + last_rows * d * 6
    eng.set_profile(False)
    eng.set_onload_policy(args.onload_policy)
    phase_b = _phase(rb0, eng.report(), K, B)

    k1 = k0  # phase D / E batches follow phase B's
    # ---- phase D (untimed): compute / transfer overlap of the next batches under CUPTI ----
    overlap, cupti_copy = None, {}
    try:
        from torch.profiler import ProfilerActivity, profile
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import kernel_times
        rd0 = eng.report()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for i in range(k1 + K, k1 + K + N_OVL):
                eng.process_batch(None, packed=packed[i])
            eng.synchronize()
            torch.cuda.synchronize()
        rd1 = eng.report()
        ov = kernel_times.overlap_stats(prof.events())
        # the KV scatter / gather kernels' own start..end (CUPTI) over the same
        # batches: CUDA-event brackets add the launch gap to these ~6-250 us kernels
        for key, tag, chunks in (("scatter", "chunk_copy_kernel<true>", rd1["onload_chunks"] - rd0["onload_chunks"]),
                                 ("gather", "chunk_copy_kernel<false>", rd1["offload_chunks"] - rd0["offload_chunks"])):
            durs = [e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
                    for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and tag in e.name]
            if durs and chunks:
                cupti_copy[key] = (sum(durs), len(durs), chunks)
        overlap = {"compute_hidden_frac": ov["compute_hidden_frac"], "h2d_busy_frac": ov["h2d_busy_frac"],
                   "batches": N_OVL,
                   "note": "CUPTI timestamps: fraction of kernel time with an H2D copy in flight; H2D engine busy "
                           "fraction of the span"}
    except Exception as e:  # profiler unavailable: the line says so
        overlap = {"unavailable": f"{type(e).__name__}: {e}"[:120]}

    # ---- phase E: the other host-hit policy on the next K batches (same engine, same
    # steady state; the control plane does not depend on the policy) ----
    alt = "always" if args.onload_policy == "adaptive" else "adaptive"
    eng.set_onload_policy(alt)
    ra0 = eng.report()
    torch.cuda.synchronize()
    ta0 = torch.cuda.Event(enable_timing=True)
    ta1 = torch.cuda.Event(enable_timing=True)
    k2 = k1 + K + N_OVL
    ta0.record()
    for i in range(k2, k2 + K):
        eng.process_batch(None, packed=packed[i])
    eng.synchronize()
    ta1.record()
    torch.cuda.synchronize()
    alt_s = ta0.elapsed_time(ta1) / 1e3
    ra1 = eng.report()
    eng.set_onload_policy(args.onload_policy)
    phase_e = _phase(ra0, ra1, K, B)

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    n_req, fresh_tokens = K * B, phase_a["fresh_tokens"]
    if dist:
        rdev = "cpu" if ONE_GPU else "cuda"
        t = torch.tensor([elapsed, e2e_s, alt_s], dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        c = torch.tensor([n_req, fresh_tokens], dtype=torch.float64, device=rdev)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        elapsed, e2e_s, alt_s = t.tolist()
        n_all, tok_all = c.tolist()
    else:
        n_all, tok_all = n_req, fresh_tokens
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    avg_launch_s = (attn_ms / 1e3) / max(attn_launches, 1)
    # DRAM traffic of one attention launch from the committed ncu capture (profiles/)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "attn_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("traffic_bytes_per_launch")
    achieved = (attn_bytes / max(attn_launches, 1)) / avg_launch_s / 1e9 if attn_launches else 0.0
    line = {
        "metric": METRIC,
        "value": n_all / elapsed,
        "unit": "requests/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": elapsed / K * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random token ids, reference-initialised random weights)",
        "config": {"workload": f"{CONFIG_TAG[args.config]} {args.config}: {cfg['L']} layers d={cfg['H'] * cfg['D']}, "
                               f"{cfg['history']}-token histories, {cfg['delta']} new + {cfg['cands']} "
                               f"candidates/request, " + (
                                   "no cache (recompute every history)" if args.mode == "recompute" else
                                   f"HBM pool {cfg['pool_frac'] * 100:g}% of users, " + (
                                       "pinned-host tier, hierarchical" if args.mode == "hierarchical"
                                       else "no host tier (gpu_only)")),
                   "mode": args.mode, "pool_frac": cfg["pool_frac"],
                   "users_per_gpu": cfg["users"], "batch": B, "device_pages": kv.device_pages,
                   "host_pinned_mb_per_rank": host_mb if hier else 0,
                   "page_size": cfg["page"], "chunk_size": cfg["chunk"], "parallelism": f"user-shard x{world}",
                   "warmup_batches_effective": warm,
                   "l2": "inputs larger than L2 (KV working set >> 126 MB)",
                   **({"host_numa_binding": numa} if numa else {}),
                   **({"host_memory_note": host_note} if host_note else {})},
        "tokens_per_sec": tok_all / elapsed,
        "p50_batch_ms": float(np.percentile(eng_lat, 50)) if eng_lat else None,
        "p99_batch_ms": float(np.percentile(eng_lat, 99)) if eng_lat else None,
        "hit_ratio": {"gpu": phase_a["gpu_hit"], "total": phase_a["total_hit"], "note": "timed phase A"},
        "phases": {"A_device": phase_a, "B_latency": phase_b, "C_e2e": phase_c, "E_other_policy": phase_e},
        "onload_policy": {
            "headline": args.onload_policy,
            "note": "host hits: 'always' onloads every persisted prefix over the host link (the reference's "
                    "executor); 'adaptive' re-encodes some on the SMs concurrently with the others' onloads. "
                    "Control plane, hit ratios and simulated clock are identical (bit-exact) under both.",
            alt: {"value": n_all / alt_s, "unit": "requests/s", "ms_per_step": alt_s / K * 1e3,
                  "h2d_GBs": phase_e["h2d_bytes_per_step"] * K / alt_s / 1e9,
                  "prefix_recomputed_frac": phase_e["prefix_recomputed_frac"], "timing": "phase E, CUDA events"},
            args.onload_policy: {"value": n_all / elapsed, "prefix_recomputed_frac": phase_a["prefix_recomputed_frac"]},
        },
        "e2e": {"value": n_all / e2e_s, "unit": "requests/s", "h2d_bytes_per_step": phase_c["h2d_bytes_per_step"],
                "d2h_bytes_per_step": phase_c["d2h_bytes_per_step"], "ms_per_step": e2e_s / K * 1e3,
                "host_wait_ms_per_step": e2e_wait / K * 1e3, "depth": depth,
                "timing": "host wall clock (perf_counter) around K pipelined submit + rankings calls, phase C"},
        "gpu_launches": int(round(launches_per_step * K)),
        "gpu_launches_per_step": launches_per_step,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak if hbm_peak else None, "traffic": traffic,
                     "traffic_source": "profiles/attn_traffic.json (ncu --set full, dram read+write bytes per launch)",
                     "kernel": "attn_tc_kernel (tcgen05 paged incremental attention)",
                     "launches_timed": attn_launches,
                     "avg_launch_us": avg_launch_s * 1e6,
                     "bytes_per_launch": attn_bytes / max(attn_launches, 1)},
        "clocks": clk,
        # host link (north star: H2D GB/s against the measured pinned-copy peak,
        # tools/probe_h2d.py: 55.5 GB/s for >= 64 MiB copies on this pool's B200 boxes)
        "host_link": {"h2d_GBs": phase_a["h2d_bytes_per_step"] * K / elapsed / 1e9, "peak_GBs": H2D_PEAK_GBS,
                      "frac": phase_a["h2d_bytes_per_step"] * K / elapsed / 1e9 / H2D_PEAK_GBS,
                      "d2h_GBs": phase_a["d2h_bytes_per_step"] * K / elapsed / 1e9,
                      "note": "timed phase A; the step is host-link bound when frac ~ 1"},
        "overlap": overlap,
        "control_plane": {"planner": args.planner,
                          "plan_ms_per_batch": float(np.mean(plan_ms)) if plan_ms else None,
                          "device_planner_kernel_us": float(np.mean(ctl_ms)) * 1e3 if args.planner == "device" else None,
                          "note": "host wall time of prepare_metadata + schedule + bookkeeping per batch (phase B)"},
    }
    # KV movement kernels (north-star "KV-gather at >= 60% of HBM roofline"): algorithmic
    # bytes = read + write of every moved chunk ([L][2][chunk][d] bf16)
    cb = kv.chunk_bytes()
    kern = {}
    for name, key, ms, ch, nl in (("chunk_scatter (onload: staging -> pages)", "scatter", copy_stat[0], copy_stat[1],
                                   copy_stat[4]),
                                  ("chunk_gather (offload: pages -> slots)", "gather", copy_stat[2], copy_stat[3],
                                   copy_stat[5])):
        if ch:
            gbs = 2 * ch * cb / (ms / 1e3) / 1e9
            kern[name] = {"achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                          "launches": nl, "avg_launch_us": ms / nl * 1e3, "bytes_per_launch": 2 * ch * cb / nl,
                          "timing": "CUDA events around each launch (phase B)"}
        if key in cupti_copy:
            us, nl2, ch2 = cupti_copy[key]
            g2 = 2 * ch2 * cb / (us / 1e6) / 1e9
            kern.setdefault(name, {})["cupti"] = {
                "achieved": g2, "frac": g2 / hbm_peak, "launches": nl2, "avg_launch_us": us / nl2,
                "bytes_per_launch": 2 * ch2 * cb / nl2, "timing": "kernel start..end timestamps (CUPTI, phase D)"}
    if proj_stat[1]:
        # projection GEMM + fused paged K/V append: read activations (rows x d) and
        # W_in (d x 4d), write u | q (rows x 2d) and the K | V append (rows x 2d), bf16
        d_ = cfg["H"] * cfg["D"]
        pbytes = proj_stat[2] * d_ * 2 * 5 + proj_stat[1] * d_ * 4 * d_ * 2
        gbs = pbytes / (proj_stat[0] / 1e3) / 1e9
        kern["gemm_tc_proj (+ fused paged K/V append)"] = {
            "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak, "launches": proj_stat[1],
            "avg_launch_us": proj_stat[0] / proj_stat[1] * 1e3, "bytes_per_launch": pbytes / proj_stat[1]}
    line["roofline"]["other_kernels"] = kern
    if args.cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, seconds=args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def cpu_baseline(cfg, seconds=15.0, threads=None):
    """The reference's own CPU serving path (oracle/_ref, value backend), all host threads."""
    from oracle.oracle import RefLib
    if not RefLib.available():
        return {"value": None, "unit": "requests/s", "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    threads = threads or os.cpu_count()
    r = RefLib().call(dict(cmd="bench", threads=threads, users_per_thread=1, history=cfg["history"],
                           delta=cfg["delta"], candidates=cfg["cands"], batch_size=1, seconds=seconds,
                           model=dict(num_layers=cfg["L"], num_heads=cfg["H"], head_dim=cfg["D"],
                                      vocab=cfg["vocab"], seed=1),
                           kv=dict(num_layers=cfg["L"], num_heads=cfg["H"], head_dim=cfg["D"],
                                   page_size=cfg["page"], chunk_size=cfg["chunk"], device_pages=4096,
                                   offload_quota=cfg["chunk"] * 64)))
    return {"value": r["requests_per_s"], "unit": "requests/s", "cores": threads, "kind": "reference",
            "sample": f"{threads} threads x 1 user each, {cfg['history']}-token prefill untimed, "
                      f"{r['requests']} revisit requests ({cfg['delta']} new + {cfg['cands']} cands) "
                      f"in {r['seconds']:.1f}s", "tokens_per_s": r["tokens_per_s"]}


def run_reference(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    base = cpu_baseline(cfg, seconds=args.cpu_seconds)
    line = {"metric": METRIC, "value": base["value"], "unit": "requests/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{CONFIG_TAG[args.config]} {args.config} (reference CPU serving path, sampled)"},
            "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": "requests/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="gr4_d256", choices=sorted(CONFIGS))
    ap.add_argument("--users", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--planner", default="host", choices=["host", "device"],
                    help="control plane: host C++ planner or the GPU (devctl.cu) lookup/LRU/victim kernel")
    ap.add_argument("--mode", default="hierarchical", choices=["hierarchical", "gpu_only", "recompute"],
                    help="configs[2] ablation: cache disabled (recompute), HBM only (gpu_only) or the hierarchical cache")
    ap.add_argument("--onload-policy", default="adaptive", choices=["always", "adaptive"],
                    help="host hits: onload every persisted prefix (the reference's executor) or re-encode some "
                         "on the SMs while others stream over the host link (same control plane)")
    ap.add_argument("--e2e-depth", type=int, default=5,
                    help="phase C: batches kept in flight before reading the oldest one's rankings (<= 5: the engine keeps 6)")
    ap.add_argument("--pool-frac", type=float, default=0.0,
                    help="configs[4] cache-pressure sweep: HBM pool as a fraction of the user population's KV")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = dict(CONFIGS[args.config])
    if args.users:
        cfg["users"] = args.users
    if args.pool_frac:
        cfg["pool_frac"] = args.pool_frac
        # configs[4]: a pool below two batches of users' pages cannot hold a
        # batch plus the users still offloading (the reference rejects it), so
        # small pools serve smaller batches instead of a silently larger pool
        ppu = -(-(cfg["history"] + 16 * cfg["delta"]) // cfg["page"])
        cfg["batch"] = max(1, min(cfg["batch"], int(args.pool_frac * cfg["users"] * ppu) // (2 * ppu)))
    world, rank, _ = dist_env()
    if world > 1 or rank != 0:
        args.cpu_baseline = False
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_b200(args, cfg)


if __name__ == "__main__":
    main()
