"""Generate tests/golden/* from the UNMODIFIED reference (oracle/_ref, built from
/root/reference by `make -C oracle ref`). Run here (the reference is not on the
GPU box); the fixtures are committed.

    python tools/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import RefLib  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def state_digest(state: dict) -> str:
    """Canonical digest of a control-plane state (tests recompute it the same way)."""
    s = dict(state)
    s["clock"] = repr(float(s["clock"]))
    return hashlib.sha256(json.dumps(s, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


CASES = [
    # (name, kv, gen or explicit trace, modes, batch sizes, backend, model)
    dict(name="alternating", backend="tag",
         kv=dict(num_layers=2, num_heads=1, head_dim=4, page_size=32, chunk_size=64, device_pages=9,
                 offload_quota=256),
         trace=[{"ts": i, "user": u, "dn": d, "nc": 1} for i, (u, d) in
                enumerate([(1, 192), (2, 192), (1, 32), (2, 32), (1, 32), (2, 32)])],
         runs=[("hierarchical", 1), ("gpu_only", 1)]),
    dict(name="gen30", backend="tag",
         kv=dict(num_layers=2, num_heads=1, head_dim=4, page_size=32, chunk_size=128, device_pages=300,
                 offload_quota=4096),
         gen=dict(num_users=30, total_requests=400, mean_final_len=600, max_len=2000, seed=12),
         runs=[("hierarchical", 4), ("gpu_only", 4), ("recompute", 4), ("hierarchical", 1)]),
    dict(name="pressure", backend="tag",
         kv=dict(num_layers=2, num_heads=1, head_dim=4, page_size=8, chunk_size=16, device_pages=48,
                 offload_quota=64),
         gen=dict(num_users=12, total_requests=300, mean_final_len=120, max_len=300, seed=404),
         runs=[("hierarchical", 3), ("gpu_only", 2)]),
    dict(name="value10", backend="value",
         kv=dict(num_layers=2, num_heads=2, head_dim=8, page_size=16, chunk_size=32, device_pages=80,
                 offload_quota=128),
         model=dict(num_layers=2, num_heads=2, head_dim=8, vocab=32, seed=4),
         gen=dict(num_users=10, total_requests=120, mean_final_len=250, min_len=10, max_len=400,
                  vocab=32, candidates=3, seed=77),
         runs=[("hierarchical", 1), ("hierarchical", 3), ("gpu_only", 1), ("recompute", 1)]),
    dict(name="value_d64", backend="value",
         kv=dict(num_layers=2, num_heads=2, head_dim=32, page_size=32, chunk_size=64, device_pages=40,
                 offload_quota=256),
         model=dict(num_layers=2, num_heads=2, head_dim=32, vocab=64, seed=9),
         gen=dict(num_users=6, total_requests=40, mean_final_len=200, min_len=50, max_len=300,
                  vocab=64, candidates=4, seed=5),
         runs=[("hierarchical", 2)]),
]


def main():
    ref = RefLib()
    os.makedirs(OUT, exist_ok=True)
    for case in CASES:
        trace = case.get("trace") or ref.gen_trace(**case["gen"])
        fixture = dict(name=case["name"], backend=case["backend"], kv=case["kv"], trace=trace,
                       model=case.get("model"), runs=[])
        for mode, bs in case["runs"]:
            req = dict(cmd="run", backend=case["backend"], kv=case["kv"], trace=trace, mode=mode,
                       batch_size=bs, check_conservation=case["backend"] == "tag")
            if case.get("model"):
                req["model"] = case["model"]
            r = ref.call(req)
            run = dict(mode=mode, batch_size=bs,
                       rejected=[b["rejected"] for b in r["batches"]],
                       digests=[state_digest(b["state"]) for b in r["batches"]],
                       final_state=r["final_state"], report=r["report"])
            if case.get("model"):
                run["logits"] = r["logits"]
            fixture["runs"].append(run)
        path = os.path.join(OUT, case["name"] + ".json")
        with open(path, "w") as f:
            json.dump(fixture, f, separators=(",", ":"))
        print(path, os.path.getsize(path))

    # generator parity: reference generate_trace output
    gens = [dict(num_users=40, total_requests=900, mean_final_len=800, max_len=3000, seed=5),
            dict(preset="mt", seed=7, total_requests=3000),
            dict(num_users=10, total_requests=300, mean_final_len=200, max_len=1000, pareto=True, seed=2),
            dict(num_users=8, total_requests=120, mean_final_len=60, max_len=200, vocab=32, candidates=3),
            dict(num_users=12, total_requests=200, mean_final_len=500, max_len=2000, fixed_delta=257)]
    out = []
    for g in gens:
        t = ref.gen_trace(**g)
        out.append(dict(gen=g, digest=hashlib.sha256(json.dumps(t, sort_keys=True).encode()).hexdigest(),
                        n=len(t), head=t[:5]))
    with open(os.path.join(OUT, "traces.json"), "w") as f:
        json.dump(out, f)

    # model forward: reference forward_incremental on a few splits (model.cpp:140)
    fw = []
    for (L, H, D, V, seed, hist_len, ncand, split) in [(2, 2, 8, 64, 5, 40, 3, 17), (1, 1, 4, 8, 1, 5, 1, 0),
                                                        (3, 2, 4, 40, 9, 30, 2, 11), (2, 2, 32, 64, 3, 100, 4, 64)]:
        import random
        rng = random.Random(seed * 100 + hist_len)
        hist = [rng.randrange(V) for _ in range(hist_len)]
        cands = [rng.randrange(V) for _ in range(ncand)]
        r = ref.call(dict(cmd="forward", model=dict(num_layers=L, num_heads=H, head_dim=D, vocab=V, seed=seed),
                          history=hist, candidates=cands, split=split))
        fw.append(dict(model=dict(num_layers=L, num_heads=H, head_dim=D, vocab=V, seed=seed), history=hist,
                       candidates=cands, split=split, logits=r["logits"], ranked=r["ranked"]))
    with open(os.path.join(OUT, "forward.json"), "w") as f:
        json.dump(fw, f)

    fp = ref.call(dict(cmd="footprint", batch=8, maxseq=40008))
    with open(os.path.join(OUT, "footprint.json"), "w") as f:
        json.dump(fp, f)
    print("done")


if __name__ == "__main__":
    main()
