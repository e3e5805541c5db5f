"""The CPU oracle (oracle/mtkv_oracle.c) pinned against the reference:
golden fixtures produced by the unmodified reference (tests/golden, see
tools/make_golden.py) and the known answers of the reference's own tests."""
import numpy as np
import pytest

from oracle.oracle import BatchRejected, ModelParams, Oracle, RefLib
from tests.util import REPORT_KEYS, batches, golden, golden_cases, state_digest


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c["name"])
def test_oracle_matches_reference_fixtures(case):
    model = ModelParams(**case["model"]) if case["model"] else None
    for run in case["runs"]:
        o = Oracle(case["kv"], mode=run["mode"], batch_size=run["batch_size"], model=model)
        logits = []
        for i, b in enumerate(batches(case["trace"], run["batch_size"])):
            rej = False
            try:
                o.process_batch(b)
            except BatchRejected:
                rej = True
            assert rej == run["rejected"][i]
            assert state_digest(o.state()) == run["digests"][i], f"{run['mode']} batch {i}"
            if model is not None and not rej:
                logits.extend(o.logits().tolist())
        o.drain()
        assert o.state() == run["final_state"]
        rep = o.report()
        for k in REPORT_KEYS:
            assert rep[k] == run["report"][k], k
        assert rep["steps_ms"] == run["report"]["steps_ms"]
        if model is not None:
            # the oracle reproduces the reference's fp64 arithmetic exactly
            assert np.array_equal(np.array(logits), np.array(run["logits"]))


def test_forward_matches_reference():
    for case in golden("forward"):
        p = ModelParams(**case["model"])
        logits, _, _ = p.forward(case["history"], case["candidates"], split=case["split"])
        assert np.array_equal(logits, np.array(case["logits"]))


def test_incremental_equals_full_random_splits():
    """test_model.cpp:133 / acceptance.cpp criterion 1: incremental == full within 1e-5."""
    rng = np.random.default_rng(17)
    p = ModelParams(2, 2, 8, 64, seed=5)
    for _ in range(25):
        hist = rng.integers(0, 64, size=int(rng.integers(1, 65))).tolist()
        cands = rng.integers(0, 64, size=int(rng.integers(1, 5))).tolist()
        split = int(rng.integers(0, len(hist) + 1))
        full, _, _ = p.forward(hist, cands, split=0)
        inc, _, _ = p.forward(hist, cands, split=split)
        assert np.abs(full - inc).max() <= 1e-5


def test_zero_weights_give_zero_logits():
    """test_model.cpp:213: SiLU(0)=0 propagates through Eq. 2-4."""
    p = ModelParams(1, 1, 4, 8, seed=1)
    for a in (p.embed, p.w_in, p.ln, p.w1, p.w2, p.w_out):
        a[:] = 0
    logits, _, _ = p.forward([1, 2], [3])
    assert (logits == 0).all()


def test_two_user_alternating_hand_oracle():
    """test_sim.cpp:75 / acceptance criterion 4(b): 768/832 total hit, 5 evictions, 64 tail tokens."""
    kv = dict(num_layers=2, num_heads=1, head_dim=4, page_size=32, chunk_size=64, device_pages=9,
              offload_quota=256)
    trace = [{"ts": i, "user": u, "dn": d, "nc": 1}
             for i, (u, d) in enumerate([(1, 192), (2, 192), (1, 32), (2, 32), (1, 32), (2, 32)])]
    o = Oracle(kv, mode="hierarchical")
    o.run(trace)
    r = o.report()
    assert r["gpu_hit_ratio"] == 0.0
    assert abs(r["total_hit_ratio"] - 768.0 / 832.0) < 1e-12
    assert r["evictions"] == 5 and r["tail_tokens_lost"] == 64
    g = Oracle(kv, mode="gpu_only")
    g.run(trace)
    assert g.report()["total_hit_ratio"] == 0.0


def test_tokens_processed_across_modes():
    """test_sim.cpp:115."""
    kv = dict(num_layers=2, num_heads=1, head_dim=4, page_size=32, chunk_size=64, device_pages=256,
              offload_quota=512)
    trace = [{"ts": i, "user": 1, "dn": 5, "nc": 1} for i in range(3)]
    reuse = Oracle(kv, mode="hierarchical")
    reuse.run(trace)
    assert reuse.report()["tokens_processed"] == 3 * 6
    re = Oracle(kv, mode="recompute")
    re.run(trace)
    assert re.report()["tokens_processed"] == 6 + 11 + 16


@pytest.mark.skipif(not RefLib.available(), reason="reference not built here")
def test_oracle_random_differential_against_reference():
    """Randomised stress (rejections, tiny pools, duplicate users in a batch)."""
    ref = RefLib()
    rng = np.random.default_rng(5)
    for _ in range(40):
        page = int(rng.choice([4, 8, 16, 32]))
        chunk = page * int(rng.choice([1, 2, 4]))
        kv = dict(num_layers=int(rng.integers(1, 4)), num_heads=1, head_dim=4, page_size=page,
                  chunk_size=chunk, device_pages=int(rng.choice([6, 12, 24, 48])),
                  offload_quota=chunk * int(rng.choice([1, 2, 4])))
        nu = int(rng.choice([2, 4, 6, 10]))
        trace = [{"ts": i, "user": int(rng.integers(nu)), "dn": int(rng.integers(0, 6 * page)),
                  "nc": int(rng.choice([1, 1, 2, page + 1]))} for i in range(40)]
        mode = str(rng.choice(["hierarchical", "gpu_only"]))
        bs = int(rng.choice([1, 2, 3, 5]))
        r = ref.call(dict(cmd="run", backend="tag", kv=kv, trace=trace, mode=mode, batch_size=bs))
        o = Oracle(kv, mode=mode, batch_size=bs)
        for i, b in enumerate(batches(trace, bs)):
            rej = False
            try:
                o.process_batch(b)
            except BatchRejected:
                rej = True
            assert rej == r["batches"][i]["rejected"]
            assert o.state() == r["batches"][i]["state"]
