"""Trace-scale control-plane parity on CPU: the host planner (the B200 engine's
serving control plane) replays the reference-generated scale fixtures
(tools/make_golden_scale.py) — the configs[1] bench stream and the reference
acceptance traces — and must reproduce the reference's complete state image
after every batch (chained digest), the drained final state and the report,
bit for bit. The GPU engine replays the same fixtures in tests/test_gpu_scale.py."""
import hashlib

import pytest

import paper_2604_22881_b200 as mtkv
from oracle.oracle import StateChain
from tests import scale_traces as st
from tests.util import REPORT_KEYS, scale_case


def _kv(case, run):
    kv = {**mtkv.KVConfig().__dict__, **case["kv"]}
    if "device_pages" in run:
        kv["device_pages"] = run["device_pages"]
    return mtkv.KVConfig(**kv)


def replay(obj, batches, run):
    ch = StateChain(run["every"])
    for b in batches:
        rej = False
        try:
            obj.process_batch(b)
        except mtkv.BatchRejected:
            rej = True
        ch.add(obj.state_blob(), rej)
    samples = ch.finish()
    n_ok = sum(a == b for a, b in zip(samples, run["chain"]))
    assert ch.n == run["n_batches"]
    # first diverging window, for the failure message
    assert samples == run["chain"], f"state diverges in batches [{64 * n_ok}, {64 * (n_ok + 1)})"
    assert ch.rejected == run["rejected"]
    obj.drain()
    assert hashlib.sha256(obj.state_blob()).hexdigest() == run["final_digest"]
    rep = obj.report()
    for k in REPORT_KEYS:
        assert rep[k] == run["report"][k], k


# bounded for the CPU suite: every fixture, the runs with <= 5000 batches
SELECT = [("scale_bench_c1", None), ("scale_c6", 5120), ("scale_c6", 81920), ("scale_c6", "recompute"),
          ("scale_c7_kuairand1k", 8), ("scale_c7_mt", 8)]


@pytest.mark.parametrize("name,pick", SELECT, ids=lambda x: str(x))
def test_host_planner_replays_reference_at_scale(name, pick):
    case = scale_case(name)
    trace, sizes = st.build(case["trace"])
    assert st.trace_digest(trace) == case["trace_digest"]
    ran = 0
    for run in case["runs"]:
        if pick == "recompute" and run["mode"] != "recompute":
            continue
        if isinstance(pick, int) and pick > 100 and run.get("device_pages") != pick:
            continue
        if isinstance(pick, int) and pick <= 100 and run["batch_size"] != pick:
            continue
        p = mtkv.Planner(_kv(case, run), mtkv.CostModel(**case["cost"]), mode=run["mode"])
        replay(p, st.split(trace, run["batch_size"], sizes), run)
        ran += 1
    assert ran > 0


@pytest.mark.parametrize("split_gbs", [(54.0, 30.0), (54.0, 3.0), (5.0, 300.0)], ids=["balanced", "slow_sms", "slow_link"])
def test_adaptive_split_keeps_reference_decisions(split_gbs):
    """The adaptive host-hit policy (planner.cpp choose_recompute, split form)
    re-encodes the earliest chunks of every host hit and onloads the rest: the
    reference's state chain, final state and report must be untouched (the same
    fixture as the 'always' replay), every host-hit prefix token must be either
    re-encoded or onloaded, chunk-aligned, and the split must follow the rates
    (slow SMs -> mostly onloaded, slow link -> mostly re-encoded)."""
    gbs, mtok = split_gbs
    case = scale_case("scale_bench_c1")
    trace, sizes = st.build(case["trace"])
    run = [r for r in case["runs"] if r["mode"] == "hierarchical"][0]
    always = mtkv.Planner(_kv(case, run), mtkv.CostModel(**case["cost"]), mode="hierarchical")
    adaptive = mtkv.Planner(_kv(case, run), mtkv.CostModel(**case["cost"]), mode="hierarchical")
    adaptive.set_onload_policy("adaptive", gbs, mtok)
    replay(adaptive, st.split(trace, run["batch_size"], sizes), run)  # bit-exact to the reference
    for b in st.split(trace, run["batch_size"], sizes):
        try:
            always.process_batch(b)
        except mtkv.BatchRejected:
            pass
    always.drain()
    ra, rb = always.report(), adaptive.report()
    chunk = case["kv"].get("chunk_size", mtkv.KVConfig().chunk_size)
    total = ra["prefix_onloaded"]
    assert ra["prefix_recomputed"] == 0 and total > 0
    assert rb["prefix_recomputed"] + rb["prefix_onloaded"] == total
    assert rb["prefix_recomputed"] % chunk == 0 and rb["prefix_onloaded"] % chunk == 0
    frac = rb["prefix_recomputed"] / total
    print(f"link {gbs} GB/s, SMs {mtok} M tok/s: re-encoded fraction {frac:.3f}")
    if mtok <= 3.0:
        assert frac < 0.2
    elif gbs <= 5.0:
        assert frac > 0.8
    else:
        assert 0.0 < frac < 1.0
