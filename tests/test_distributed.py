"""N>1 path on CPU (gloo, world_size 2): users shard by id across ranks, each
rank owns an independent cache shard, the only cross-rank traffic is the
timing/count reduction bench.py does (no collective on the data path)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_2604_22881_b200 as mtkv
    cfg = dict(bench.CONFIGS["tiny_d64"], users=48, history=256, batch=8)
    prefill, revisits = bench.make_workload(cfg, n_batches=12, rank=rank, world=world)
    users = sorted({r["user"] for r in prefill} | {r["user"] for r in revisits})
    from paper_2604_22881_b200.shard import shard_of
    assert all(shard_of(u, world) == rank for u in users)  # user-id hash sharding
    kv = bench.kv_config(cfg)
    p = mtkv.Planner(kv, mtkv.CostModel(bus_bandwidth=55e9))
    for i in range(0, len(prefill), 4):
        p.process_batch(prefill[i:i + 4])
    for i in range(0, len(revisits), cfg["batch"]):
        p.process_batch(revisits[i:i + cfg["batch"]])
    r = p.report()
    # a shard run alone is the same run: decisions depend on the shard only
    q = mtkv.Planner(kv, mtkv.CostModel(bus_bandwidth=55e9))
    for i in range(0, len(prefill), 4):
        q.process_batch(prefill[i:i + 4])
    for i in range(0, len(revisits), cfg["batch"]):
        q.process_batch(revisits[i:i + cfg["batch"]])
    assert q.state() == p.state()
    t = torch.tensor([r["requests"], r["hist_required"], r["hist_device"] + r["hist_host"]], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    mx = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    gathered = [None] * world
    dist.all_gather_object(gathered, users)
    if rank == 0:
        out.put((t.tolist(), mx.item(), gathered, r["requests"]))
    dist.barrier()
    dist.destroy_process_group()


def test_user_sharding_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    totals, mx, gathered, r0_requests = q.get()
    assert mx == 2.0
    assert not (set(gathered[0]) & set(gathered[1]))           # disjoint shards
    assert totals[0] == 2 * (48 + 12 * 8)                       # every request served once
    assert totals[2] <= totals[1]


def _shard_worker(rank, world, port, out):
    """One rank = one cache shard: it sees the global request stream, keeps the
    requests of its users (shard.local_requests, no collective), and its control
    plane must reproduce the reference run on its sub-trace bit for bit."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import hashlib
    import paper_2604_22881_b200 as mtkv
    from oracle.oracle import StateChain
    from paper_2604_22881_b200.shard import local_requests
    from tests import scale_traces as st
    from tests.util import scale_case
    case = scale_case("scale_shards")
    run = [r for r in case["runs"] if r["shards"] == world and r["shard"] == rank][0]
    trace, _ = st.build(case["trace"])
    kv = mtkv.KVConfig(**{**mtkv.KVConfig().__dict__, **case["kv"]})
    p = mtkv.Planner(kv, mode="hierarchical")
    ch = StateChain(run["every"])
    mine = 0
    for i in range(0, len(trace), case["batch"]):
        sub = local_requests(trace[i:i + case["batch"]], rank, world)
        if sub:
            p.process_batch(sub)
            ch.add(p.state_blob())
            mine += len(sub)
    p.drain()
    ok = (ch.finish() == run["chain"] and ch.n == run["n_batches"]
          and hashlib.sha256(p.state_blob()).hexdigest() == run["final_digest"])
    t = torch.tensor([float(mine), float(ok)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    if rank == 0:
        out.put((t.tolist(), len(trace)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_trace_matches_reference_per_shard_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=600)
        assert pr.exitcode == 0
    (served, ok), n = q.get()
    assert served == n          # every request served by exactly one shard
    assert ok == world          # every shard bit-identical to the reference on its sub-trace
