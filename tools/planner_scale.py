"""Control-plane cost per batch, host planner vs device planner, as the user
population and the batch grow. Tag backend with a one-layer
d=16 model so the data plane is negligible; requests are revisits drawn
uniformly from the population with a pool of ~5 % of it, so every batch
evicts. One JSON line per (users, batch, planner).

  python tools/planner_scale.py [--batches 40]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_22881_b200 as mtkv  # noqa: E402


def run(users: int, batch: int, planner: str, batches: int, hist: int = 256, delta: int = 32) -> dict:
    page = 16
    ppu = -(-(hist + batches * delta) // page)
    kv = mtkv.KVConfig(num_layers=1, num_heads=1, head_dim=16, page_size=page, chunk_size=64,
                       device_pages=max(int(0.05 * users * (hist // page)), 4 * batch * ppu),
                       onload_pages=batch * ppu + 64, offload_quota=64 * 4 * batch)
    eng = mtkv.Engine(kv, mode="hierarchical", backend="tag", batch_size=batch, planner=planner,
                      max_users=users + 64, max_user_pages=ppu + 64, host_reserve_mb=0)
    rng = np.random.default_rng(0)
    ts = 0
    for i in range(0, users, batch):  # first visits
        eng.process_batch([{"ts": ts + j, "user": u, "dn": hist, "nc": 1} for j, u in enumerate(range(i, min(users, i + batch)))])
        ts += batch
    eng.synchronize()
    plan_ms, kern_ms = [], []
    t0 = time.perf_counter()
    for b in range(batches):
        us = rng.choice(users, size=batch, replace=False)
        eng.process_batch([{"ts": ts + j, "user": int(u), "dn": delta, "nc": 1} for j, u in enumerate(us)])
        ts += batch
        pm, km = eng.last_plan_ms()
        plan_ms.append(pm)
        kern_ms.append(km)
    eng.synchronize()
    wall = time.perf_counter() - t0
    rep = eng.report()
    return {"users": users, "batch": batch, "planner": planner, "plan_ms_per_batch": float(np.mean(plan_ms)),
            "plan_ms_p90": float(np.percentile(plan_ms, 90)),
            "device_kernel_ms": float(np.mean(kern_ms)) if planner == "device" else None,
            "wall_ms_per_batch": wall / batches * 1e3, "evictions": rep["evictions"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=40)
    args = ap.parse_args()
    # (65536 users / batch 512 exhausted the box's host memory for the pinned tier)
    for users, batch in ((2048, 64), (16384, 256)):
        for planner in ("host", "device"):
            print(json.dumps(run(users, batch, planner, args.batches)), flush=True)


if __name__ == "__main__":
    main()
