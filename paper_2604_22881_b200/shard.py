"""User-id sharding of the serving path across GPUs (north star: "requests shard
naturally by user-id hash across the 8 GPUs of one box, each GPU owning an
independent cache shard, so there are no collectives on the hot path").

A user's whole state (its pages in one GPU's HBM pool, its chunks in that
GPU's pinned host tier, its LRU position) lives on exactly one shard, so a
request never needs another shard's data: the router splits every batch by
`shard_of(user)`, each shard runs its own engine on its sub-batch (same
relative order, so each shard sees exactly the reference engine's behaviour on
its sub-trace), and rankings are gathered back in request order.

* `shard_of(user, n)` — the shard function: a 32-bit integer mixer (the
  murmur3 finaliser) of the user id, mod n. Stable across processes and runs.
* `Router` — splits a batch into per-shard sub-batches and merges per-shard
  results back into request order.
* `ShardedEngine` — N engines in one process (one per GPU, or several on one
  GPU for functional checks): submit / rankings like `Engine`.
* `local_requests` — the torchrun form: every rank sees the request stream and
  keeps its own users (no collective on the data path).
"""
from __future__ import annotations

from typing import Sequence


def shard_of(user: int, n: int) -> int:
    """murmur3 fmix32 of the user id, mod n."""
    if n <= 1:
        return 0
    h = int(user) & 0xFFFFFFFF
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & 0xFFFFFFFF
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & 0xFFFFFFFF
    h ^= h >> 16
    return h % n


class Router:
    def __init__(self, n: int):
        if n < 1:
            raise ValueError("need at least one shard")
        self.n = n

    def split(self, batch: Sequence[dict]):
        """-> (sub-batches per shard, [(shard, index in its sub-batch)] per request)"""
        subs = [[] for _ in range(self.n)]
        where = []
        for r in batch:
            s = shard_of(r["user"], self.n)
            where.append((s, len(subs[s])))
            subs[s].append(r)
        return subs, where

    @staticmethod
    def merge(where, per_shard):
        """per-shard result lists -> one list in request order"""
        return [per_shard[s][i] for s, i in where]


def local_requests(batch: Sequence[dict], rank: int, world: int) -> list:
    """The rank's share of a batch (torchrun: one engine per rank)."""
    return [r for r in batch if shard_of(r["user"], world) == rank]


class ShardedEngine:
    """N independent cache shards behind one submit / rankings interface."""

    def __init__(self, engines: Sequence):
        self.engines = list(engines)
        self.router = Router(len(self.engines))

    def process_batch(self, batch: Sequence[dict]) -> None:
        subs, self._where = self.router.split(batch)
        for eng, sub in zip(self.engines, subs):
            if sub:
                eng.process_batch(sub)
        self._subs = subs

    def last_rankings(self) -> list:
        per = [eng.last_rankings() if sub else [] for eng, sub in zip(self.engines, self._subs)]
        return Router.merge(self._where, per)

    def submit(self, batch: Sequence[dict]):
        subs, where = self.router.split(batch)
        tickets = [eng.submit(sub) if sub else None for eng, sub in zip(self.engines, subs)]
        return where, tickets

    def rankings(self, handle) -> list:
        where, tickets = handle
        per = [eng.rankings(t) if t is not None else [] for eng, t in zip(self.engines, tickets)]
        return Router.merge(where, per)

    def drain(self) -> None:
        for eng in self.engines:
            eng.drain()

    def reports(self) -> list:
        return [eng.report() for eng in self.engines]
