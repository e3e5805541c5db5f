"""BASELINE.json configs[2] and configs[4] on one B200 (one JSON object per line).

  python tools/sweep.py ablation   # configs[2]: recompute vs gpu_only vs hierarchical, same trace
  python tools/sweep.py pressure   # configs[4]: HBM pool 2%..50% of the working set

Both use bench.py's workload (configs[1] model: 4 layers, d=256, 4K-token
histories, 64 new tokens + 8 candidates per request, lognormal revisits) and
time the device with CUDA events over K batches after a warm-up; the per-mode
numbers are the same metric as bench.py (requests/s, tokens/s, p50/p99 batch ms,
hit ratios, host-link bytes), plus the compute/transfer overlap of a CUPTI
replay of the timed batches (fraction of kernel time with an H2D copy in flight). Multi-GPU points are bench.py under torchrun
(user-sharded, no collective: every rank runs this exact per-GPU workload).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def run_mode(cfg: dict, mode: str, steps: int, warm: int, pool_frac: float | None = None) -> dict:
    import torch
    import paper_2604_22881_b200 as mtkv
    cfg = dict(cfg)
    if pool_frac is not None:
        cfg["pool_frac"] = pool_frac
    kv = bench.kv_config(cfg)
    model = mtkv.ModelConfig(num_layers=cfg["L"], num_heads=cfg["H"], head_dim=cfg["D"], vocab=cfg["vocab"], seed=1)
    B = cfg["batch"]
    n_extra = 16  # fresh batches after the timed ones: 8 profiled (overlap), 8 for per-batch latency
    prefill, revisits = bench.make_workload(cfg, warm + steps + n_extra, 0, 1)
    tok = kv.token_kv_bytes()
    extent_mb = -(-((cfg["history"] + 16 * cfg["delta"]) * tok) // 2**20)
    host_mb = int(1.1 * cfg["users"] * extent_mb) + 1024 if mode == "hierarchical" else 0
    eng = mtkv.Engine(kv, mtkv.CostModel(bus_bandwidth=55e9), mode=mode, backend="value", batch_size=B,
                      model=model, host_reserve_mb=host_mb, host_extent_mb=extent_mb)
    if mode != "recompute":  # recompute keeps no cache: the first visit is not a prefill
        pb = max(1, min(cfg["batch"], 65536 // cfg["history"]))
        for i in range(0, len(prefill), pb):
            eng.process_batch(prefill[i:i + pb])
    else:  # the recompute engine still needs each user's token history
        for i in range(0, len(prefill), 4):
            eng.process_batch(prefill[i:i + 4])
    batches = [mtkv.RequestBatch(revisits[i * B:(i + 1) * B]) for i in range(warm + steps + n_extra)]
    for i in range(warm):
        eng.process_batch(None, packed=batches[i])
    eng.synchronize()
    r0 = eng.report()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for i in range(warm, warm + steps):
        eng.process_batch(None, packed=batches[i])
    eng.synchronize()
    t1.record()
    torch.cuda.synchronize()
    el = t0.elapsed_time(t1) / 1e3
    r1 = eng.report()
    ph = bench._phase(r0, r1, steps, B)
    # compute/transfer overlap under CUPTI (tools/kernel_times.overlap_stats) on the
    # next 8 batches of the same stream (fresh requests, not a replay)
    from torch.profiler import ProfilerActivity, profile
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import kernel_times
    tb = warm + steps
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(tb, tb + 8):
            eng.process_batch(None, packed=batches[i])
        eng.synchronize()
        torch.cuda.synchronize()
    ov = kernel_times.overlap_stats(prof.events())
    # per-batch latency (enqueue -> done, one batch in flight) on the 8 after those
    eng.set_profile(True)
    lat = []
    for i in range(tb + 8, tb + 16):
        eng.process_batch(None, packed=batches[i])
        eng.synchronize()
        lat.append(eng.last_batch_ms())
    return {"mode": mode, "pool_frac": cfg["pool_frac"], "device_pages": kv.device_pages, "users": cfg["users"],
            "batch": B, "requests_per_s": steps * B / el, "tokens_processed_per_request": ph["fresh_tokens"] / (steps * B),
            "fresh_tokens_per_s": ph["fresh_tokens"] / el, "ms_per_batch": el / steps * 1e3,
            "p50_batch_ms": float(np.percentile(lat, 50)), "p99_batch_ms": float(np.percentile(lat, 99)),
            "gpu_hit": ph["gpu_hit"], "total_hit": ph["total_hit"],
            "h2d_GBs": ph["h2d_bytes_per_step"] * steps / el / 1e9,
            "h2d_busy_frac": ph["h2d_bytes_per_step"] * steps / el / 55.5e9,
            "evictions": ph["evictions"],
            "overlap": {"compute_hidden_frac": ov["compute_hidden_frac"], "h2d_busy_frac_cupti": ov["h2d_busy_frac"],
                        "note": "CUPTI, 8 batches after the timed ones: fraction of kernel time with an H2D copy in flight"}}


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "ablation"
    cfg = dict(bench.CONFIGS["gr4_d256"])
    out = []
    if what == "ablation":
        cfg["users"] = 512
        for mode in ("hierarchical", "gpu_only", "recompute"):
            out.append({"config": "configs[2] recompute-vs-reuse", **run_mode(cfg, mode, steps=12, warm=24)})
            print(json.dumps(out[-1]), flush=True)
    elif what == "pressure":
        cfg["batch"] = 16
        for frac in (0.02, 0.05, 0.10, 0.20, 0.50):
            out.append({"config": "configs[4] cache-pressure", **run_mode(cfg, "hierarchical", steps=24, warm=48,
                                                                          pool_frac=frac)})
            print(json.dumps(out[-1]), flush=True)
    else:
        raise SystemExit(__doc__)


if __name__ == "__main__":
    main()
