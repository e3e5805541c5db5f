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
    assert all(u % world == rank for u in users)  # user-id sharding
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
