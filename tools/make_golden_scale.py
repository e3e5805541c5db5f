"""Trace-scale parity fixtures from the UNMODIFIED reference (oracle/_ref):
tests/golden/scale_*.json. Run here (the reference is not on the GPU box):

    python tools/make_golden_scale.py

Every run stores the chained digest of the reference's complete control-plane
state image after every batch (oracle.oracle.StateChain, sampled every 64
batches), the rejected batches, the digest of the drained final state and the
reference's RunReport. tests/test_gpu_scale.py replays the same traces through
the B200 engine (tag backend: every byte moved is checked by the conservation
read-back) with the host planner and with the device planner.

Cases:
  scale_bench_c1    the exact configs[1] request stream bench.py serves in the
                    driver's run (2048 users x 4096-token prefill, 113 revisit
                    batches of 64, pool 10 %, page 32, chunk 128), model
                    geometry L=4 H=2 D=128 (the simulated clock charges bytes)
  scale_c6          reference acceptance criterion 6 (tests/acceptance.cpp:283):
                    kuairand1k seed 1, L=2 H=1 D=4, DevicePages 5120..81920,
                    hierarchical batch 4, plus recompute
  scale_c7          criterion 7 (tests/acceptance.cpp:314): kuairand1k and mt
                    seed 1, batch 1/4/8 x recompute/gpu_only/hierarchical
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import RefLib  # noqa: E402
from tests import scale_traces as st  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
SMALL_KV = dict(num_layers=2, num_heads=1, head_dim=4)  # acceptance.cpp:287-290


def cases():
    c1kv = st.bench_kv("gr4_d256")
    yield dict(name="scale_bench_c1", trace=dict(kind="bench", config="gr4_d256", n_batches=113),
               kv=c1kv, cost=dict(bus_bandwidth=55e9),
               runs=[dict(mode="hierarchical", batch_size=64), dict(mode="gpu_only", batch_size=64)])
    yield dict(name="scale_c6", trace=dict(kind="preset", preset="kuairand1k", seed=1), kv=SMALL_KV, cost={},
               runs=[dict(mode="hierarchical", batch_size=4, device_pages=p) for p in (5120, 10240, 20480, 40960, 81920)]
               + [dict(mode="recompute", batch_size=4)])
    for preset in ("kuairand1k", "mt"):
        yield dict(name=f"scale_c7_{preset}", trace=dict(kind="preset", preset=preset, seed=1), kv=SMALL_KV, cost={},
                   runs=[dict(mode=m, batch_size=b) for b in (1, 4, 8) for m in ("hierarchical", "gpu_only", "recompute")])


def shard_fixture(ref):
    """scale_shards: the kuairand1k trace (criterion 6 geometry, pool 5120 pages,
    batch 8) routed over N = 2 and 4 user-id shards (paper_2604_22881_b200.shard):
    the reference run on each shard's sub-trace, with the sub-batches the router
    produces from the global batches."""
    from paper_2604_22881_b200.shard import Router
    spec = dict(kind="preset", preset="kuairand1k", seed=1)
    trace, _ = st.build(spec)
    kv = dict(SMALL_KV, device_pages=5120)
    fx = dict(name="scale_shards", trace=spec, trace_digest=st.trace_digest(trace), kv=kv, cost={}, batch=8,
              runs=[])
    for n in (2, 4):
        router = Router(n)
        subs = [[] for _ in range(n)]
        sizes = [[] for _ in range(n)]
        for i in range(0, len(trace), 8):
            parts, _ = router.split(trace[i:i + 8])
            for s_, part in enumerate(parts):
                if part:
                    subs[s_].extend(part)
                    sizes[s_].append(len(part))
        for s_ in range(n):
            req = dict(cmd="run", backend="tag", kv=kv, cost={}, trace=subs[s_], mode="hierarchical",
                       batch_size=8, batch_sizes=sizes[s_])
            r = ref.run_blobs(req, every=64)
            fx["runs"].append(dict(shards=n, shard=s_, mode="hierarchical", batch_size=8, **r))
            print("scale_shards", n, s_, r["n_batches"], "gpu_hit %.4f" % r["report"]["gpu_hit_ratio"], flush=True)
    with open(os.path.join(OUT, "scale_shards.json"), "w") as f:
        json.dump(fx, f, separators=(",", ":"))


def main(only=None):
    ref = RefLib()
    if not only or "scale_shards" in only:
        shard_fixture(ref)
    for case in cases():
        if only and case["name"] not in only:
            continue
        t0 = time.time()
        trace, sizes = st.build(case["trace"])
        fx = dict(name=case["name"], trace=case["trace"], trace_digest=st.trace_digest(trace), n_requests=len(trace),
                  kv=case["kv"], cost=case["cost"], runs=[])
        for run in case["runs"]:
            kv = dict(case["kv"])
            if "device_pages" in run:
                kv["device_pages"] = run["device_pages"]
            req = dict(cmd="run", backend="tag", kv=kv, cost=case["cost"], trace=trace, mode=run["mode"],
                       batch_size=run["batch_size"])
            if sizes:
                req["batch_sizes"] = sizes
            r = ref.run_blobs(req, every=64)
            fx["runs"].append(dict(run, **r))
            print(case["name"], run, r["n_batches"], "rejected", len(r["rejected"]),
                  "gpu_hit %.4f" % r["report"]["gpu_hit_ratio"], "%.1fs" % (time.time() - t0), flush=True)
        with open(os.path.join(OUT, case["name"] + ".json"), "w") as f:
            json.dump(fx, f, separators=(",", ":"))


if __name__ == "__main__":
    main(set(sys.argv[1:]) or None)
