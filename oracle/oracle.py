"""ctypes bindings for the CPU checkers. TEST INFRASTRUCTURE ONLY.

* ``Oracle``  — the C restatement (oracle/mtkv_oracle.c, built by ``make -C oracle oracle``).
* ``RefLib``  — the unmodified reference compiled in place (oracle/_ref, ``make -C oracle ref``);
  present only where /root/reference was available at build time (the .so travels).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg import this module.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
from typing import Iterable

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libmtkv_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmtkv_ref.so")

MODES = {"recompute": 0, "gpu_only": 1, "hierarchical": 2}
KV_FIELDS = ["num_layers", "num_heads", "head_dim", "page_size", "chunk_size", "device_pages",
             "onload_pages", "bytes_per_element", "offload_quota", "host_capacity"]
COST_FIELDS = ["bus_bandwidth", "tx_setup", "host_bandwidth", "page_op", "attn_coeff",
               "linear_coeff", "embed_coeff", "layout_coeff", "meta_fixed", "strip_fixed",
               "embed_fixed", "layout_fixed", "await_fixed", "update_fixed", "commit_per_chunk",
               "offload_submit", "post_fixed"]


class KV(C.Structure):
    _fields_ = [(f, C.c_uint32) for f in KV_FIELDS[:8]] + [("offload_quota", C.c_uint64),
                                                           ("host_capacity", C.c_uint64)]


class Cost(C.Structure):
    _fields_ = [(f, C.c_double) for f in COST_FIELDS]


class Model(C.Structure):
    _fields_ = [("num_layers", C.c_uint32), ("num_heads", C.c_uint32), ("head_dim", C.c_uint32),
                ("vocab", C.c_uint32)] + [(n, C.POINTER(C.c_double)) for n in
                                          ("embed", "w_in", "ln", "w1", "w2", "w_out")]


class Plan(C.Structure):
    _fields_ = [("user", C.c_uint32), ("history_len", C.c_uint64), ("reusable_len", C.c_uint64),
                ("device_served", C.c_uint64), ("host_onload", C.c_uint64),
                ("fresh_history", C.c_uint64), ("delta", C.c_uint32),
                ("num_candidates", C.c_uint32), ("onload_chunks", C.c_uint32),
                ("scratch_pages", C.c_uint32)]


class Eviction(C.Structure):
    _fields_ = [("user", C.c_uint32), ("freed_pages", C.c_uint64), ("tail_tokens_lost", C.c_uint64)]


class UserState(C.Structure):
    _fields_ = [("total_len", C.c_uint64), ("device_len", C.c_uint64), ("persisted_len", C.c_uint64),
                ("last_access", C.c_uint64), ("locked", C.c_uint32), ("num_pages", C.c_uint32),
                ("host_chunks", C.c_uint32), ("pending_offload", C.c_uint32)]


class Report(C.Structure):
    _fields_ = [("step_ms", C.c_double * 9), ("wait_ms", C.c_double), ("comp_ms", C.c_double),
                ("gpu_hit_ratio", C.c_double), ("total_hit_ratio", C.c_double),
                ("tokens_processed", C.c_uint64), ("evictions", C.c_uint64),
                ("tail_tokens_lost", C.c_uint64), ("requests", C.c_uint64), ("batches", C.c_uint64),
                ("avg_latency_ms", C.c_double), ("total_latency_ms", C.c_double),
                ("peak_pages", C.c_uint64), ("pages_allocated", C.c_uint64),
                ("occupied_pages", C.c_uint64), ("free_pages", C.c_uint64),
                ("quota_in_flight", C.c_uint64), ("clock", C.c_double)]


STEP_LABELS = ["Step 1-2. Prepare Metadata", "Step 3. Strip Tokens", "Step 4. Embedding",
               "Step 5. Data Layout", "Step 6. Await Metadata", "Step 7. Update Metadata",
               "Step 8. HSTU Inference", "Step 9. Offload KV", "Step 10. Postprocess"]

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
        L = C.CDLL(ORACLE_SO)
        L.orc_engine_new.restype = C.c_void_p
        L.orc_engine_new.argtypes = [C.POINTER(KV), C.POINTER(Cost), C.c_int, C.c_uint32, C.c_int,
                                     C.POINTER(Model)]
        L.orc_engine_free.argtypes = [C.c_void_p]
        u32p, u64p = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
        L.orc_process_batch.argtypes = [C.c_void_p, C.c_uint32, u64p, u32p, u32p, u32p, u32p, u32p]
        L.orc_drain.argtypes = [C.c_void_p]
        L.orc_last_error.restype = C.c_char_p
        L.orc_last_error.argtypes = [C.c_void_p]
        L.orc_last_plans.restype = C.c_uint32
        L.orc_last_plans.argtypes = [C.c_void_p, C.POINTER(Plan), C.c_uint32]
        L.orc_last_evictions.restype = C.c_uint32
        L.orc_last_evictions.argtypes = [C.c_void_p, C.POINTER(Eviction), C.c_uint32]
        L.orc_last_logits.restype = C.c_uint32
        L.orc_last_logits.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_uint32]
        L.orc_known_users.restype = C.c_uint32
        L.orc_known_users.argtypes = [C.c_void_p, u32p, C.c_uint32]
        L.orc_user_state_get.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(UserState)]
        L.orc_user_pages.restype = C.c_uint32
        L.orc_user_pages.argtypes = [C.c_void_p, C.c_uint32, u32p, C.c_uint32]
        L.orc_lru_snapshot.restype = C.c_uint32
        L.orc_lru_snapshot.argtypes = [C.c_void_p, u32p, C.c_uint32]
        L.orc_report_get.argtypes = [C.c_void_p, C.POINTER(Report)]
        L.orc_evict_user.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_is_locked.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_model_random.argtypes = [C.c_uint32] * 4 + [C.c_uint64] + [C.POINTER(C.c_double)] * 6
        L.orc_forward.argtypes = [C.POINTER(Model), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                  C.c_uint64, u32p, C.c_uint32, u32p, C.c_uint32,
                                  C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _lib = L
    return _lib


def default_kv(**over) -> dict:
    kv = dict(num_layers=8, num_heads=4, head_dim=128, page_size=32, chunk_size=1024,
              device_pages=40960, onload_pages=10008, bytes_per_element=2, offload_quota=8192,
              host_capacity=0)
    kv.update(over)
    return kv


def default_cost(**over) -> dict:
    c = dict(bus_bandwidth=25e9, tx_setup=10e-6, host_bandwidth=50e9, page_op=50e-9,
             attn_coeff=2e-10, linear_coeff=1e-7, embed_coeff=5e-8, layout_coeff=5e-8,
             meta_fixed=1e-4, strip_fixed=5e-5, embed_fixed=1e-4, layout_fixed=1e-4,
             await_fixed=5e-5, update_fixed=5e-5, commit_per_chunk=5e-6, offload_submit=3e-5,
             post_fixed=2e-4)
    c.update(over)
    return c


class ModelParams:
    """Reference weight init (model.cpp:34) reproduced bit-for-bit by the C oracle."""

    def __init__(self, num_layers, num_heads, head_dim, vocab, seed=1):
        import numpy as np
        d = num_heads * head_dim
        self.cfg = dict(num_layers=num_layers, num_heads=num_heads, head_dim=head_dim, vocab=vocab,
                        seed=seed)
        self.embed = np.zeros(vocab * d)
        self.w_in = np.zeros(num_layers * d * 4 * d)
        self.ln = np.zeros(num_layers * d)
        self.w1 = np.zeros(num_layers * d * d)
        self.w2 = np.zeros(num_layers * d * d)
        self.w_out = np.zeros(d * vocab)
        dp = C.POINTER(C.c_double)
        lib().orc_model_random(num_layers, num_heads, head_dim, vocab, seed,
                               *[a.ctypes.data_as(dp) for a in (self.embed, self.w_in, self.ln,
                                                                 self.w1, self.w2, self.w_out)])
        self.struct = Model(num_layers, num_heads, head_dim, vocab,
                            *[a.ctypes.data_as(dp) for a in (self.embed, self.w_in, self.ln,
                                                              self.w1, self.w2, self.w_out)])

    def forward(self, history, candidates, split=0, cached_k=None, cached_v=None):
        import numpy as np
        hist = np.asarray(history, dtype=np.uint32)
        cands = np.asarray(candidates, dtype=np.uint32)
        L, d = self.cfg["num_layers"], self.cfg["num_heads"] * self.cfg["head_dim"]
        logits = np.zeros(self.cfg["vocab"])
        u32p, dp = C.POINTER(C.c_uint32), C.POINTER(C.c_double)
        ck = cv = None
        if split > 0:
            if cached_k is None:
                M = split + 1
                wk, wv = np.zeros(L * M * d), np.zeros(L * M * d)
                tmp = np.zeros(self.cfg["vocab"])
                pre = np.ascontiguousarray(hist[:split])
                one = np.zeros(1, dtype=np.uint32)
                lib().orc_forward(C.byref(self.struct), None, None, 0, pre.ctypes.data_as(u32p),
                                  split, one.ctypes.data_as(u32p), 1, tmp.ctypes.data_as(dp),
                                  wk.ctypes.data_as(dp), wv.ctypes.data_as(dp))
                cached_k = np.ascontiguousarray(wk.reshape(L, M, d)[:, :split])
                cached_v = np.ascontiguousarray(wv.reshape(L, M, d)[:, :split])
            ck, cv = cached_k.ctypes.data_as(dp), cached_v.ctypes.data_as(dp)
        delta = np.ascontiguousarray(hist[split:])
        M = len(delta) + len(cands)
        nk, nv = np.zeros(L * M * d), np.zeros(L * M * d)
        rc = lib().orc_forward(C.byref(self.struct), ck, cv, split, delta.ctypes.data_as(u32p),
                               len(delta), cands.ctypes.data_as(u32p), len(cands),
                               logits.ctypes.data_as(dp), nk.ctypes.data_as(dp),
                               nv.ctypes.data_as(dp))
        if rc != 0:
            raise ValueError("forward: token id out of vocabulary or no candidates")
        return logits, nk.reshape(L, M, d), nv.reshape(L, M, d)


class OracleError(RuntimeError):
    pass


class BatchRejected(OracleError):
    pass


def _batch_arrays(batch):
    import numpy as np
    n = len(batch)
    ts = np.array([r.get("ts", 0) for r in batch], dtype=np.uint64)
    users = np.array([r["user"] for r in batch], dtype=np.uint32)
    dn = np.array([len(r["tokens"]) if r.get("tokens") else r["dn"] for r in batch], dtype=np.uint32)
    nc = np.array([len(r["cands"]) if r.get("cands") else r["nc"] for r in batch], dtype=np.uint32)
    toks = np.array([t for r in batch for t in (r.get("tokens") or [])] or [0], dtype=np.uint32)
    cands = np.array([t for r in batch for t in (r.get("cands") or [])] or [0], dtype=np.uint32)
    return n, ts, users, dn, nc, toks, cands


class Oracle:
    """C-oracle engine with the same per-batch state dump as the reference driver."""

    def __init__(self, kv: dict, mode="hierarchical", batch_size=1, cost: dict | None = None,
                 model: ModelParams | None = None):
        self.kvd = default_kv(**kv)
        self.kv = KV(**self.kvd)
        self.cost = Cost(**default_cost(**(cost or {})))
        self.model = model
        self.batch_size = batch_size
        self.h = lib().orc_engine_new(C.byref(self.kv), C.byref(self.cost), MODES[mode], batch_size,
                                      1 if model else 0, C.byref(model.struct) if model else None)
        if not self.h:
            raise OracleError("invalid configuration")

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_engine_free(self.h)
            self.h = None

    def process_batch(self, batch):
        import numpy as np
        n, ts, users, dn, nc, toks, cands = _batch_arrays(batch)
        u32p, u64p = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
        rc = lib().orc_process_batch(self.h, n, ts.ctypes.data_as(u64p), users.ctypes.data_as(u32p),
                                     dn.ctypes.data_as(u32p), nc.ctypes.data_as(u32p),
                                     toks.ctypes.data_as(u32p), cands.ctypes.data_as(u32p))
        if rc == 2:
            raise BatchRejected(lib().orc_last_error(self.h).decode())
        if rc != 0:
            raise OracleError(lib().orc_last_error(self.h).decode())

    def run(self, trace, per_batch=None):
        out = []
        for i in range(0, len(trace), self.batch_size):
            b = trace[i:i + self.batch_size]
            rej = False
            try:
                self.process_batch(b)
            except BatchRejected:
                rej = True
            out.append({"rejected": rej, **(per_batch(self) if per_batch else {})})
        self.drain()
        return out

    def drain(self):
        lib().orc_drain(self.h)

    def plans(self):
        n = lib().orc_last_plans(self.h, None, 0)
        arr = (Plan * max(n, 1))()
        lib().orc_last_plans(self.h, arr, n)
        return [{f: getattr(arr[i], f) for f, _ in Plan._fields_} for i in range(n)]

    def evictions(self):
        n = lib().orc_last_evictions(self.h, None, 0)
        arr = (Eviction * max(n, 1))()
        lib().orc_last_evictions(self.h, arr, n)
        return [{f: getattr(arr[i], f) for f, _ in Eviction._fields_} for i in range(n)]

    def logits(self):
        import numpy as np
        if not self.model:
            return None
        n = lib().orc_last_logits(self.h, None, 0)
        out = np.zeros((max(n, 1), self.model.cfg["vocab"]))
        lib().orc_last_logits(self.h, out.ctypes.data_as(C.POINTER(C.c_double)), n)
        return out[:n]

    def evict_user(self, user):
        if lib().orc_evict_user(self.h, user) != 0:
            raise OracleError(lib().orc_last_error(self.h).decode())

    def is_locked(self, user):
        return bool(lib().orc_is_locked(self.h, user))

    def report(self):
        r = Report()
        lib().orc_report_get(self.h, C.byref(r))
        d = {f: getattr(r, f) for f, _ in Report._fields_ if f != "step_ms"}
        d["steps_ms"] = dict(zip(STEP_LABELS, list(r.step_ms)))
        return d

    def state(self):
        """Same schema as ref_driver.cpp dump_state()."""
        n = lib().orc_known_users(self.h, None, 0)
        ids = (C.c_uint32 * max(n, 1))()
        lib().orc_known_users(self.h, ids, n)
        users = []
        for i in range(n):
            u = ids[i]
            s = UserState()
            lib().orc_user_state_get(self.h, u, C.byref(s))
            np_ = lib().orc_user_pages(self.h, u, None, 0)
            pg = (C.c_uint32 * max(np_, 1))()
            lib().orc_user_pages(self.h, u, pg, np_)
            users.append(dict(user=u, total_len=s.total_len, device_len=s.device_len,
                              persisted_len=s.persisted_len, locked=bool(s.locked),
                              last_access=s.last_access, pages=list(pg)[:np_],
                              host_chunks=s.host_chunks, pending_offload=s.pending_offload))
        m = lib().orc_lru_snapshot(self.h, None, 0)
        lru = (C.c_uint32 * max(m, 1))()
        lib().orc_lru_snapshot(self.h, lru, m)
        r = self.report()
        return dict(users=users, lru=list(lru)[:m], evictions=r["evictions"],
                    tail_tokens_lost=r["tail_tokens_lost"], pages_allocated=r["pages_allocated"],
                    occupied_pages=r["occupied_pages"], free_pages=r["free_pages"],
                    quota_in_flight=r["quota_in_flight"], clock=r["clock"])


class RefLib:
    """The unmodified reference (oracle/_ref); JSON in / JSON out."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.L = C.CDLL(path)
        self.L.mtkv_ref_call.restype = C.c_void_p
        self.L.mtkv_ref_call.argtypes = [C.c_char_p]
        self.L.mtkv_ref_free.argtypes = [C.c_void_p]

    @staticmethod
    def available(path=REF_SO) -> bool:
        return os.path.exists(path)

    def call(self, req: dict) -> dict:
        p = self.L.mtkv_ref_call(json.dumps(req).encode())
        s = C.string_at(p).decode()
        self.L.mtkv_ref_free(p)
        out = json.loads(s)
        if "error" in out:
            raise OracleError(out["error"])
        return out

    def run_blobs(self, req: dict, every: int = 64) -> dict:
        """"run" with per-batch canonical state images (mtkv_state_blob layout)
        hashed on the fly: returns the chained digest (see state_chain) sampled
        every `every` batches, the rejected batch indices, the drained final
        state's digest and the report."""
        import hashlib
        CB = C.CFUNCTYPE(None, C.c_uint64, C.POINTER(C.c_uint8), C.c_uint64, C.c_int)
        if not hasattr(self.L, "_rb"):
            self.L.mtkv_ref_run_blobs.restype = C.c_void_p
            self.L.mtkv_ref_run_blobs.argtypes = [C.c_char_p, CB]
            self.L._rb = True
        chain = StateChain(every)
        final = {}

        def cb(i, data, n, rejected):
            blob = C.string_at(data, n)
            if i == 2**64 - 1:
                final["digest"] = hashlib.sha256(blob).hexdigest()
            else:
                chain.add(blob, bool(rejected))

        fn = CB(cb)
        p = self.L.mtkv_ref_run_blobs(json.dumps(req).encode(), fn)
        s = C.string_at(p).decode()
        self.L.mtkv_ref_free(p)
        out = json.loads(s)
        if "error" in out:
            raise OracleError(out["error"])
        return dict(chain=chain.finish(), every=every, n_batches=chain.n, rejected=chain.rejected,
                    final_digest=final["digest"], report=out["report"])

    def gen_trace(self, **gen) -> list:
        out = self.call({"cmd": "gen_trace", **gen})
        return [json.loads(line) for line in out["jsonl"].splitlines() if line.strip()]


class StateChain:
    """Chained digest of per-batch state images: c_0 = 32 zero bytes,
    c_i = sha256(c_{i-1} || sha256(blob_i)); c_i is sampled at every `every`-th
    batch and at the last one, so a divergence is located to an `every`-batch
    window while the fixture stays small. Shared by the fixture generator and
    the GPU replay tests (tests/test_gpu_scale.py)."""

    def __init__(self, every: int = 64):
        self.every, self.n, self.c = every, 0, bytes(32)
        self.samples, self.rejected = [], []

    def add(self, blob: bytes, rejected: bool = False) -> None:
        import hashlib
        self.c = hashlib.sha256(self.c + hashlib.sha256(blob).digest()).digest()
        if rejected:
            self.rejected.append(self.n)
        self.n += 1
        if self.n % self.every == 0:
            self.samples.append(self.c.hex())

    def finish(self) -> list:
        if self.n % self.every:
            self.samples.append(self.c.hex())
        return self.samples


def load_jsonl(path) -> list:
    with open(path) as f:
        return [json.loads(x) for x in f if x.strip()]
