"""In-situ kernel durations of the serving step (CUPTI activity timestamps via torch.profiler).

Runs bench.py's configs[1] workload (same engine setup as tools/sweep.py), then
records `--steps` pipelined batches under torch.profiler and prints one JSON
line per kernel name: launches, mean/min/max device duration in us. Unlike the
engine's CUDA-event brackets these are the kernel's own start/end timestamps,
and unlike an ncu launch list the kernels run concurrently with the copy
engines exactly as in the bench.

  python tools/kernel_times.py [--steps 8] [--warm 24] [--config gr4_d256]
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _union(iv):
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def overlap_stats(events) -> dict:
    """Compute/transfer overlap over a profiled window (torch.profiler CUDA
    events): the fraction of device compute time (union of kernel intervals)
    that ran while a host->device copy was in flight, and how busy the H2D
    engine was. compute_hidden_frac ~ 1 means the onload traffic fully overlaps
    the compute (or, when the link is the bottleneck, the compute is hidden).
    Kernel time outside [first copy start, last copy end] — the pipeline drain
    after the window's last onload — is not counted (it has no next batch's
    copy to hide behind)."""
    import torch
    cuda = [e for e in events if e.device_type == torch.autograd.DeviceType.CUDA]
    h = _union([(e.time_range.start, e.time_range.end) for e in cuda if "HtoD" in e.name])
    h_lo, h_hi = (h[0][0], h[-1][1]) if h else (0.0, 0.0)
    k = _union([(max(e.time_range.start, h_lo), min(e.time_range.end, h_hi)) for e in cuda
                if not e.name.startswith("Memcpy") and not e.name.startswith("Memset")
                and e.time_range.end > h_lo and e.time_range.start < h_hi])
    inter, j = 0.0, 0
    for a, b in k:
        while j < len(h) and h[j][1] <= a:
            j += 1
        jj = j
        while jj < len(h) and h[jj][0] < b:
            inter += max(0.0, min(b, h[jj][1]) - max(a, h[jj][0]))
            jj += 1
    kb = sum(b - a for a, b in k)
    hb = sum(b - a for a, b in h)
    return {"compute_busy_us": kb, "h2d_busy_us": hb, "span_us": h_hi - h_lo,
            "compute_hidden_frac": inter / kb if kb else None,
            "h2d_busy_frac": hb / (h_hi - h_lo) if h_hi > h_lo else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warm", type=int, default=24)
    ap.add_argument("--config", default="gr4_d256")
    ap.add_argument("--users", type=int, default=0)
    ap.add_argument("--trace", default="", help="also write a chrome trace (JSON) here")
    ap.add_argument("--ncu", action="store_true", help="bracket the measured batches with cudaProfilerStart/Stop "
                    "(run under ncu --profile-from-start off) instead of torch.profiler")
    ap.add_argument("--policy", default="adaptive", choices=["adaptive", "always"], help="host-hit onload policy")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    import paper_2604_22881_b200 as mtkv
    cfg = dict(bench.CONFIGS[args.config])
    if args.users:
        cfg["users"] = args.users
    kv = bench.kv_config(cfg)
    model = mtkv.ModelConfig(num_layers=cfg["L"], num_heads=cfg["H"], head_dim=cfg["D"], vocab=cfg["vocab"], seed=1)
    B = cfg["batch"]
    prefill, revisits = bench.make_workload(cfg, args.warm + args.steps, 0, 1)
    tok = kv.token_kv_bytes()
    extent_mb = -(-((cfg["history"] + 16 * cfg["delta"]) * tok) // 2**20)
    eng = mtkv.Engine(kv, mtkv.CostModel(bus_bandwidth=55e9), mode="hierarchical", backend="value", batch_size=B,
                      model=model, host_reserve_mb=int(1.1 * cfg["users"] * extent_mb) + 1024,
                      host_extent_mb=extent_mb, onload_policy=args.policy)
    pb = max(1, min(cfg["batch"], 65536 // cfg["history"]))
    for i in range(0, len(prefill), pb):
        eng.process_batch(prefill[i:i + pb])
    batches = [mtkv.RequestBatch(revisits[i * B:(i + 1) * B]) for i in range(args.warm + args.steps)]
    for i in range(args.warm):
        eng.process_batch(None, packed=batches[i])
    eng.synchronize()
    torch.cuda.synchronize()
    if args.ncu:  # ncu --profile-from-start off: only the measured batches are captured
        torch.cuda.profiler.start()
        for i in range(args.warm, args.warm + args.steps):
            eng.process_batch(None, packed=batches[i])
        eng.synchronize()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(args.warm, args.warm + args.steps):
            eng.process_batch(None, packed=batches[i])
        eng.synchronize()
        torch.cuda.synchronize()
    if args.trace:
        prof.export_chrome_trace(args.trace)
    dur = collections.defaultdict(list)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            dur[ev.name].append(ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total)
    # per batch: the layer stack's device span, embed start -> scoring kernel end
    # (PDL-launched kernels start early and wait, so their own durations overlap
    # their predecessors'; the span is the honest per-batch compute time)
    kev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
                 key=lambda e: e.time_range.start)
    spans, t_embed = [], None
    for e in kev:
        if "embed_kernel" in e.name:
            t_embed = e.time_range.start
        elif "pick_scores" in e.name and t_embed is not None:
            spans.append(e.time_range.end - t_embed)
            t_embed = None
    print(json.dumps({"overlap": overlap_stats(prof.events())}), flush=True)
    if spans:
        print(json.dumps({"layer_stack_span_us": {"mean": sum(spans) / len(spans), "min": min(spans),
                                                  "max": max(spans), "batches": len(spans)}}), flush=True)
    rows = sorted(dur.items(), key=lambda kv_: -sum(kv_[1]))
    for name, d in rows:
        print(json.dumps({"kernel": name[:90], "n": len(d), "per_step": len(d) / args.steps,
                          "mean_us": sum(d) / len(d), "min_us": min(d), "max_us": max(d),
                          "share_us_per_step": sum(d) / args.steps}), flush=True)


if __name__ == "__main__":
    main()
