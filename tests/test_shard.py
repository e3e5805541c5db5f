"""Router / ShardedEngine host logic (CPU) and the in-process sharded engine on
the GPU (several shards on GPU 0): per-shard state equals the reference run on
the shard's sub-trace (tests/golden/scale_shards.json)."""
import hashlib

import pytest

import paper_2604_22881_b200 as mtkv
from oracle.oracle import StateChain
from paper_2604_22881_b200.shard import Router, ShardedEngine, local_requests, shard_of
from tests import scale_traces as st
from tests.util import scale_case


def test_shard_function_is_stable_and_balanced():
    assert [shard_of(u, 8) for u in range(8)] == [shard_of(u, 8) for u in range(8)]
    assert shard_of(12345, 1) == 0
    counts = [0] * 8
    for u in range(80000):
        counts[shard_of(u, 8)] += 1
    assert max(counts) / min(counts) < 1.03


def test_router_split_merge_round_trip():
    batch = [{"user": u, "i": i} for i, u in enumerate([5, 9, 5, 1, 77, 9, 3])]
    r = Router(3)
    subs, where = r.split(batch)
    assert sum(len(s) for s in subs) == len(batch)
    for s_, sub in enumerate(subs):
        assert all(shard_of(x["user"], 3) == s_ for x in sub)
        assert [x["i"] for x in sub] == sorted(x["i"] for x in sub)  # order kept within a shard
        assert sub == local_requests(batch, s_, 3)
    assert Router.merge(where, [[x["i"] for x in sub] for sub in subs]) == list(range(len(batch)))


class _PlannerShard:
    """Host planner with the engine's submit/rankings-free surface (CPU)."""

    def __init__(self, kv):
        self.p = mtkv.Planner(kv, mode="hierarchical")
        self.chain = StateChain(64)

    def process_batch(self, b):
        self.p.process_batch(b)
        self.chain.add(self.p.state_blob())

    def drain(self):
        self.p.drain()

    def report(self):
        return self.p.report()


def _check_shards(shards, case, n):
    runs = sorted([r for r in case["runs"] if r["shards"] == n], key=lambda r: r["shard"])
    for sh, run in zip(shards, runs):
        assert sh.chain.finish() == run["chain"] and sh.chain.n == run["n_batches"]
        blob = sh.p.state_blob() if hasattr(sh, "p") else sh.eng.state_blob()
        assert hashlib.sha256(blob).hexdigest() == run["final_digest"]


def test_sharded_planners_match_reference_per_shard():
    case = scale_case("scale_shards")
    trace, _ = st.build(case["trace"])
    kv = mtkv.KVConfig(**{**mtkv.KVConfig().__dict__, **case["kv"]})
    shards = [_PlannerShard(kv) for _ in range(2)]
    se = ShardedEngine(shards)
    for i in range(0, len(trace), case["batch"]):
        se.process_batch(trace[i:i + case["batch"]])
    se.drain()
    _check_shards(shards, case, 2)


class _EngineShard:
    def __init__(self, kv):
        self.eng = mtkv.Engine(kv, mode="hierarchical", backend="tag", batch_size=8)
        self.chain = StateChain(64)

    def process_batch(self, b):
        self.eng.process_batch(b)
        self.chain.add(self.eng.state_blob())

    def drain(self):
        self.eng.drain()

    def report(self):
        return self.eng.report()


@pytest.mark.gpu
def test_sharded_gpu_engines_match_reference_per_shard():
    case = scale_case("scale_shards")
    trace, _ = st.build(case["trace"])
    kv = mtkv.KVConfig(**{**mtkv.KVConfig().__dict__, **case["kv"]})
    shards = [_EngineShard(kv) for _ in range(4)]
    se = ShardedEngine(shards)
    for i in range(0, len(trace), case["batch"]):
        se.process_batch(trace[i:i + case["batch"]])
    se.drain()
    _check_shards(shards, case, 4)
    for sh in shards:
        sh.eng.check_conservation()
