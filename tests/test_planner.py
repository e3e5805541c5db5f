"""The product's host control plane (paper_2604_22881_b200 Planner, C-ABI) is
bit-exact with the reference: every decision of every batch (hit class,
evictions, page ids, locks, persisted lengths, simulated clock) on the golden
traces, plus randomized differential tests against the C oracle."""
import random

import pytest

import paper_2604_22881_b200 as mtkv
from oracle.oracle import BatchRejected as OracleRejected, Oracle
from tests.util import REPORT_KEYS, batches, golden_cases, state_digest


def _kv(d):
    return mtkv.KVConfig(**{**mtkv.KVConfig().__dict__, **d})


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c["name"])
def test_planner_matches_reference_fixtures(case):
    for run in case["runs"]:
        p = mtkv.Planner(_kv(case["kv"]), mode=run["mode"])
        for i, b in enumerate(batches(case["trace"], run["batch_size"])):
            rej = False
            try:
                p.process_batch(b)
            except mtkv.BatchRejected:
                rej = True
            assert rej == run["rejected"][i]
            assert state_digest(p.state()) == run["digests"][i], f"{case['name']} {run['mode']} batch {i}"
        p.drain()
        assert p.state() == run["final_state"]
        rep = p.report()
        for k in REPORT_KEYS:
            assert rep[k] == run["report"][k], k
        assert rep["steps_ms"] == run["report"]["steps_ms"]


def _compare_plans(p, o):
    assert p.plans() == o.plans()
    assert p.evictions() == o.evictions()


def test_planner_random_differential_with_evict_pressure():
    """acceptance.cpp criterion 8-style interleavings: batches, drains and
    external evictions, compared decision-by-decision against the oracle;
    safety properties checked after every event."""
    rng = random.Random(404)
    kv = dict(num_layers=2, num_heads=1, head_dim=4, page_size=8, chunk_size=16, device_pages=48,
              offload_quota=64)
    for sched in range(60):
        p = mtkv.Planner(_kv(kv), mode="hierarchical")
        o = Oracle(kv, mode="hierarchical")
        ts = 0
        for _ in range(80):
            op = rng.randrange(4)
            if op < 2:
                b = []
                for _ in range(1 + rng.randrange(3)):
                    b.append({"ts": ts, "user": rng.randrange(6), "dn": 1 + rng.randrange(30), "nc": 1})
                    ts += 1
                e1 = e2 = None
                try:
                    p.process_batch(b)
                except mtkv.BatchRejected as e:
                    e1 = e
                try:
                    o.process_batch(b)
                except OracleRejected as e:
                    e2 = e
                assert (e1 is None) == (e2 is None)
                if e1 is None:
                    _compare_plans(p, o)
            elif op == 2:
                p.drain()
                o.drain()
            else:
                users = p.known_users()
                if not users:
                    continue
                u = users[rng.randrange(len(users))]
                locked = p.is_locked(u)
                assert locked == o.is_locked(u)
                if locked:
                    with pytest.raises(mtkv.Error):
                        p.evict_user(u)  # (a) locked users are never evicted
                else:
                    p.evict_user(u)
                    o.evict_user(u)
            st = p.state()
            assert st == o.state()
            r = p.report()
            assert r["quota_in_flight"] <= kv["offload_quota"]                    # (b)
            assert r["occupied_pages"] + r["free_pages"] == kv["device_pages"]    # (c)


def test_lru_order_matches_naive_reference():
    """test_manager.cpp:274 / criterion 9: recency order == naive list, evictions from the tail."""
    rng = random.Random(99)
    kv = _kv(dict(num_layers=1, num_heads=1, head_dim=4, page_size=4, chunk_size=4, device_pages=4096,
                  offload_quota=4))
    p = mtkv.Planner(kv, mode="gpu_only")
    naive = []
    for i in range(3000):
        u = rng.randrange(50)
        if rng.random() < 0.7:
            p.process_batch([{"ts": i, "user": u, "dn": 1, "nc": 1}])
            if u in naive:
                naive.remove(u)
            naive.insert(0, u)
        elif u in p.known_users():
            p.evict_user(u)
            if u in naive:
                naive.remove(u)
        assert p.lru_snapshot() == naive


def test_locking_protocol_and_rejections():
    """test_manager.cpp:431 locking protocol / :457 oversized batches."""
    kv = _kv(dict(num_layers=2, page_size=8, chunk_size=16, device_pages=4, offload_quota=64))
    p = mtkv.Planner(kv, mode="hierarchical")
    with pytest.raises(mtkv.BatchRejected):
        p.process_batch([{"user": 1, "dn": 100, "nc": 1}])
    with pytest.raises(mtkv.Error):
        p.process_batch([{"user": 2, "dn": 1, "nc": 0}])


def test_zero_copy_eviction_keeps_persisted_prefix():
    """test_manager.cpp:393: evicting a user frees its pages without transfers;
    the persisted prefix survives and is onloaded on the next visit."""
    kv = _kv(dict(num_layers=2, num_heads=1, head_dim=4, page_size=8, chunk_size=16, device_pages=64,
                  offload_quota=64))
    p = mtkv.Planner(kv, mode="hierarchical")
    p.process_batch([{"user": 5, "dn": 40, "nc": 1}])
    p.drain()  # two chunks persisted
    st = p.user_state(5)
    assert st["persisted_len"] == 32 and st["device_len"] == 40
    before = p.report()
    p.evict_user(5)
    after = p.report()
    assert after["tail_tokens_lost"] - before["tail_tokens_lost"] == 8
    assert p.get_total_cache_length(5) == 32
    p.process_batch([{"user": 5, "dn": 10, "nc": 1}])
    plan = p.plans()[0]
    assert plan["history_len"] == 40 and plan["host_onload"] == 32
    assert plan["onload_chunks"] == 2 and plan["fresh_history"] == 8
