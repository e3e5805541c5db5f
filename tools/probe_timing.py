"""Timing probe on bench.py's configs[1] workload (diagnostics, not a bench line).

  python tools/probe_timing.py [--steps 16] [--warm 24]

1. device throughput (phase A style) under each host-hit policy;
2. end-to-end public-API throughput (submit / rankings) at pipeline depths 1-3;
3. the attention launch timed three ways on the same batches: CUDA-event
   brackets (bench phase B), CUPTI start..end of the same bracketed launches,
   and CUPTI of unbracketed (PDL-chained) launches.
One JSON object per line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--warm", type=int, default=24)
    ap.add_argument("--config", default="gr4_d256")
    ap.add_argument("--sequence", default="probe", choices=["probe", "bench", "host"])
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    import paper_2604_22881_b200 as mtkv
    cfg = dict(bench.CONFIGS[args.config])
    kv = bench.kv_config(cfg)
    model = mtkv.ModelConfig(num_layers=cfg["L"], num_heads=cfg["H"], head_dim=cfg["D"], vocab=cfg["vocab"], seed=1)
    B, K = cfg["batch"], args.steps
    n_b = args.warm + 12 * K
    prefill, revisits = bench.make_workload(cfg, n_b, 0, 1)
    tok = kv.token_kv_bytes()
    extent_mb = -(-((cfg["history"] + 16 * cfg["delta"]) * tok) // 2**20)
    ppu = -(-(cfg["history"] + 16 * cfg["delta"]) // cfg["page"])
    eng = mtkv.Engine(kv, mtkv.CostModel(bus_bandwidth=55e9), mode="hierarchical", backend="value", batch_size=B,
                      model=model, host_reserve_mb=int(1.1 * cfg["users"] * extent_mb) + 1024,
                      host_extent_mb=extent_mb, max_users=cfg["users"] + 64, max_user_pages=2 * ppu + 64,
                      onload_policy="adaptive")
    pb = max(1, min(B, 65536 // cfg["history"]))
    for i in range(0, len(prefill), pb):
        eng.process_batch(prefill[i:i + pb])
    batches = [revisits[i * B:(i + 1) * B] for i in range(n_b)]
    packed = [mtkv.RequestBatch(b) for b in batches]
    for i in range(args.warm):
        eng.process_batch(None, packed=packed[i])
    eng.synchronize()
    cur = args.warm

    def take(n):
        nonlocal cur
        r = range(cur, cur + n)
        cur += n
        return r

    def e2e(depth, tag):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pending, wait_s = [], 0.0
        for i in take(K):
            pending.append(eng.submit(batches[i]))
            if len(pending) > depth:
                w0 = time.perf_counter()
                eng.rankings(pending.pop(0))
                wait_s += time.perf_counter() - w0
        for t in pending:
            eng.rankings(t)
        eng.synchronize()
        dt = time.perf_counter() - t0
        print(json.dumps({"probe": "e2e", "at": tag, "depth": depth, "req_s": K * B / dt, "ms_per_step": dt / K * 1e3,
                          "host_wait_ms_per_step": wait_s / K * 1e3}), flush=True)

    def device(pol, tag):
        eng.set_onload_policy(pol)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in take(K):
            eng.process_batch(None, packed=packed[i])
        eng.synchronize()
        dt = time.perf_counter() - t0
        eng.set_onload_policy("adaptive")
        print(json.dumps({"probe": "device", "at": tag, "policy": pol, "req_s": K * B / dt,
                          "ms_per_step": dt / K * 1e3}), flush=True)

    if args.sequence == "host":  # host-side cost per call: packing, submit, rankings, process_batch
        import numpy as np
        pk, sb, rk, pbt = [], [], [], []
        for i in take(K):
            t0 = time.perf_counter()
            eng.process_batch(None, packed=packed[i])
            pbt.append(time.perf_counter() - t0)
        eng.synchronize()
        pending = []
        for i in take(K):
            t0 = time.perf_counter()
            rb = mtkv.RequestBatch(batches[i])
            t1 = time.perf_counter()
            pending.append(eng.submit(packed=rb))
            t2 = time.perf_counter()
            pk.append(t1 - t0)
            sb.append(t2 - t1)
            if len(pending) > 2:
                t3 = time.perf_counter()
                eng.rankings(pending.pop(0))
                rk.append(time.perf_counter() - t3)
        for t in pending:
            eng.rankings(t)
        eng.synchronize()
        ms = lambda v: round(float(np.median(v)) * 1e3, 3)
        print(json.dumps({"probe": "host_ms_median", "process_batch": ms(pbt), "pack": ms(pk), "submit": ms(sb),
                          "rankings_wait": ms(rk), "process_batch_p90": round(float(np.percentile(pbt, 90)) * 1e3, 3)}),
              flush=True)
        return

    if args.sequence == "bench":  # bench.py's phase order: A, B (sync, always, profile), C, E
        device("adaptive", "A")
        e2e(2, "after A")
        eng.set_onload_policy("always")
        eng.set_profile(True)
        for i in take(K):
            eng.process_batch(None, packed=packed[i])
            eng.synchronize()
        eng.set_profile(False)
        eng.set_onload_policy("adaptive")
        e2e(2, "after B")
        device("adaptive", "after B")
        device("always", "after B")
        eng.set_profile(True)
        device("adaptive", "profile on")
        eng.set_profile(False)
        device("adaptive", "profile off again")
        return

    # 1. device throughput per policy
    for pol in ("adaptive", "always"):
        eng.set_onload_policy(pol)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in take(K):
            eng.process_batch(None, packed=packed[i])
        eng.synchronize()
        dt = time.perf_counter() - t0
        print(json.dumps({"probe": "device", "policy": pol, "req_s": K * B / dt, "ms_per_step": dt / K * 1e3}),
              flush=True)
    eng.set_onload_policy("adaptive")

    # 2. e2e through submit / rankings at several pipeline depths
    for depth in (3, 4, 5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pending, wait_s = [], 0.0
        for i in take(K):
            pending.append(eng.submit(batches[i]))
            if len(pending) > depth:
                w0 = time.perf_counter()
                eng.rankings(pending.pop(0))
                wait_s += time.perf_counter() - w0
        for t in pending:
            eng.rankings(t)
        eng.synchronize()
        dt = time.perf_counter() - t0
        print(json.dumps({"probe": "e2e", "depth": depth, "req_s": K * B / dt, "ms_per_step": dt / K * 1e3,
                          "host_wait_ms_per_step": wait_s / K * 1e3}), flush=True)

    # 3. attention timing: event brackets vs CUPTI (same launches), then CUPTI without brackets
    def attn_cupti(prof):
        return [e.device_time_total for e in prof.events()
                if e.device_type == torch.autograd.DeviceType.CUDA and "attn_tc_kernel" in e.name]

    eng.set_onload_policy("always")
    eng.set_profile(True)
    ev_ms, ev_n = 0.0, 0
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in take(K):
            eng.process_batch(None, packed=packed[i])
            eng.synchronize()
            ms, n = eng.last_attention_ms()
            ev_ms += ms
            ev_n += n
        torch.cuda.synchronize()
    d = attn_cupti(prof)
    print(json.dumps({"probe": "attn_bracketed", "event_avg_us": ev_ms / max(ev_n, 1) * 1e3, "launches": ev_n,
                      "cupti_avg_us": sum(d) / max(len(d), 1), "cupti_n": len(d),
                      "cupti_min_us": min(d) if d else None, "cupti_max_us": max(d) if d else None}), flush=True)
    eng.set_profile(False)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in take(K):
            eng.process_batch(None, packed=packed[i])
            eng.synchronize()
        torch.cuda.synchronize()
    d = attn_cupti(prof)
    print(json.dumps({"probe": "attn_pdl_chained", "cupti_avg_us": sum(d) / max(len(d), 1), "cupti_n": len(d),
                      "cupti_min_us": min(d) if d else None, "cupti_max_us": max(d) if d else None}), flush=True)


if __name__ == "__main__":
    main()
