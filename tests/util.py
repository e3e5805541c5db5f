"""Shared helpers for the parity tests."""
import glob
import hashlib
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def state_digest(state: dict) -> str:
    """Same canonicalisation as tools/make_golden.py."""
    s = dict(state)
    s["clock"] = repr(float(s["clock"]))
    return hashlib.sha256(json.dumps(s, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


def golden(name: str) -> dict:
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)


def golden_cases(backend=None):
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "*.json"))):
        name = os.path.basename(p)[:-5]
        if name in ("traces", "forward", "footprint") or name.startswith("scale_"):
            continue
        g = golden(name)
        if backend is None or g["backend"] == backend:
            out.append(g)
    return out


REPORT_KEYS = ["gpu_hit_ratio", "total_hit_ratio", "tokens_processed", "evictions", "tail_tokens_lost",
               "requests", "batches", "avg_latency_ms", "total_latency_ms", "peak_pages", "wait_ms", "comp_ms"]


def batches(trace, bs):
    return [trace[i:i + bs] for i in range(0, len(trace), bs)]


def scale_case(name: str) -> dict:
    return golden(name)


SCALE_CASES = ["scale_bench_c1", "scale_c6", "scale_c7_kuairand1k", "scale_c7_mt"]
