"""B200-native hierarchical user-KV-cache serving path (MTServe hot path).

Python mirror of the reference's C++ serving API (``mtkv::Engine<B>``,
``mtkv::CacheManager``, ``generate_trace``; /root/reference/proj/core/include/mtkv)
over the C-ABI library ``libmtkv_b200.so`` (include/mtkv_b200.h). Same names,
argument meaning and error behaviour: ``Error`` where the reference throws
``mtkv::Error``, ``BatchRejected`` where it throws ``mtkv::BatchRejected``.

The GPU engine has no CPU fallback: constructing an ``Engine`` without a usable
CUDA device raises ``NoDevice``. ``Planner`` is the host control plane only
(decisions, no payloads) and works anywhere.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field, asdict
from typing import Iterable, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmtkv_b200.so")

MODE = {"recompute": 0, "gpu_only": 1, "hierarchical": 2}
BACKEND = {"tag": 0, "value": 1}
STEP_LABELS = ["Step 1-2. Prepare Metadata", "Step 3. Strip Tokens", "Step 4. Embedding",
               "Step 5. Data Layout", "Step 6. Await Metadata", "Step 7. Update Metadata",
               "Step 8. HSTU Inference", "Step 9. Offload KV", "Step 10. Postprocess"]


class Error(RuntimeError):
    """mtkv::Error (core.hpp:16)."""


class BatchRejected(Error):
    """mtkv::BatchRejected (manager.hpp:76)."""


class NoDevice(Error):
    """No usable CUDA device: the B200 engine refuses to run (no CPU fallback)."""


# ----------------------------------------------------------------- structs ---
class _KV(C.Structure):
    _fields_ = [(f, C.c_uint32) for f in ("num_layers", "num_heads", "head_dim", "page_size",
                                          "chunk_size", "device_pages", "onload_pages",
                                          "bytes_per_element")] + \
               [("offload_quota", C.c_uint64), ("host_capacity", C.c_uint64)]


_COST_FIELDS = ["bus_bandwidth", "tx_setup", "host_bandwidth", "page_op", "attn_coeff",
                "linear_coeff", "embed_coeff", "layout_coeff", "meta_fixed", "strip_fixed",
                "embed_fixed", "layout_fixed", "await_fixed", "update_fixed", "commit_per_chunk",
                "offload_submit", "post_fixed"]


class _Cost(C.Structure):
    _fields_ = [(f, C.c_double) for f in _COST_FIELDS]


class _ModelCfg(C.Structure):
    _fields_ = [("num_layers", C.c_uint32), ("num_heads", C.c_uint32), ("head_dim", C.c_uint32),
                ("vocab", C.c_uint32), ("seed", C.c_uint64)]


class _Request(C.Structure):
    _fields_ = [("timestamp", C.c_uint64), ("user", C.c_uint32), ("new_token_count", C.c_uint32),
                ("candidate_count", C.c_uint32), ("new_tokens", C.POINTER(C.c_uint32)),
                ("candidates", C.POINTER(C.c_uint32))]


class _Plan(C.Structure):
    _fields_ = [("user", C.c_uint32), ("history_len", C.c_uint64), ("reusable_len", C.c_uint64),
                ("device_served", C.c_uint64), ("host_onload", C.c_uint64),
                ("fresh_history", C.c_uint64), ("delta", C.c_uint32), ("num_candidates", C.c_uint32),
                ("onload_chunks", C.c_uint32), ("scratch_pages", C.c_uint32)]


class _Eviction(C.Structure):
    _fields_ = [("user", C.c_uint32), ("freed_pages", C.c_uint64), ("tail_tokens_lost", C.c_uint64)]


class _SeqState(C.Structure):
    _fields_ = [("total_len", C.c_uint64), ("device_len", C.c_uint64), ("persisted_len", C.c_uint64),
                ("last_access", C.c_uint64), ("locked", C.c_uint32), ("num_pages", C.c_uint32),
                ("host_chunks", C.c_uint32), ("pending_offload", C.c_uint32)]


class _Report(C.Structure):
    _fields_ = [("step_ms", C.c_double * 9), ("wait_ms", C.c_double), ("comp_ms", C.c_double),
                ("gpu_hit_ratio", C.c_double), ("total_hit_ratio", C.c_double),
                ("tokens_processed", C.c_uint64), ("evictions", C.c_uint64),
                ("tail_tokens_lost", C.c_uint64), ("requests", C.c_uint64), ("batches", C.c_uint64),
                ("avg_latency_ms", C.c_double), ("total_latency_ms", C.c_double),
                ("peak_pages", C.c_uint64), ("pages_allocated", C.c_uint64),
                ("occupied_pages", C.c_uint64), ("free_pages", C.c_uint64),
                ("quota_in_flight", C.c_uint64), ("clock", C.c_double), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("onload_chunks", C.c_uint64),
                ("offload_chunks", C.c_uint64), ("hist_required", C.c_uint64),
                ("hist_device", C.c_uint64), ("hist_host", C.c_uint64),
                ("prefix_onloaded", C.c_uint64), ("prefix_recomputed", C.c_uint64)]


class _EngineOpts(C.Structure):
    _fields_ = [("mode", C.c_int), ("backend", C.c_int), ("batch_size", C.c_uint32),
                ("seed", C.c_uint64), ("model", _ModelCfg), ("device", C.c_int),
                ("max_batch_tokens", C.c_uint32), ("max_user_pages", C.c_uint32),
                ("keep_logits", C.c_uint32), ("profile", C.c_uint32), ("host_reserve_mb", C.c_uint64),
                ("device_planner", C.c_uint32), ("max_users", C.c_uint32), ("host_extent_mb", C.c_uint32),
                ("onload_policy", C.c_uint32), ("onload_gbs", C.c_double), ("recompute_mtok_s", C.c_double)]


class _GenCfg(C.Structure):
    _fields_ = [("num_users", C.c_uint32), ("total_requests", C.c_uint64), ("pareto", C.c_int),
                ("gap_log_mu", C.c_double), ("gap_log_sigma", C.c_double),
                ("pareto_alpha", C.c_double), ("pareto_scale_ms", C.c_double),
                ("mean_final_len", C.c_double), ("min_len", C.c_uint64), ("max_len", C.c_uint64),
                ("fixed_delta", C.c_uint32), ("candidates", C.c_uint32), ("vocab", C.c_uint32),
                ("seed", C.c_uint64)]


EXPORTED_SYMBOLS = [
    "mtkv_kv_config_default", "mtkv_kv_config_validate", "mtkv_parse_config_text",
    "mtkv_cost_model_default", "mtkv_pages_needed", "mtkv_persisted_prefix", "mtkv_last_error",
    "mtkv_planner_create", "mtkv_planner_destroy", "mtkv_planner_process_batch", "mtkv_planner_drain",
    "mtkv_planner_set_onload_policy",
    "mtkv_planner_prepare_metadata", "mtkv_planner_scratch_pages", "mtkv_planner_release_scratch",
    "mtkv_planner_commit_onload", "mtkv_planner_finish_append", "mtkv_planner_advance_persisted",
    "mtkv_planner_lock_user", "mtkv_planner_unlock_user", "mtkv_planner_last_page_len",
    "mtkv_engine_create", "mtkv_engine_destroy", "mtkv_engine_process_batch", "mtkv_engine_run",
    "mtkv_engine_drain", "mtkv_engine_synchronize", "mtkv_engine_last_logits",
    "mtkv_engine_last_rankings", "mtkv_engine_batch_rankings", "mtkv_engine_batches_submitted",
    "mtkv_engine_last_plan_ms",
    "mtkv_engine_check_conservation", "mtkv_engine_read_user_kv",
    "mtkv_engine_last_batch_ms", "mtkv_engine_last_attention_ms", "mtkv_engine_last_chunk_copy_ms",
    "mtkv_engine_last_proj_ms",
    "mtkv_engine_kernel_launches",
    "mtkv_engine_set_profile", "mtkv_engine_set_onload_policy",
    "mtkv_report", "mtkv_last_plans", "mtkv_last_evictions", "mtkv_known_users", "mtkv_user_state",
    "mtkv_user_pages", "mtkv_lru_snapshot", "mtkv_evict_user", "mtkv_is_locked",
    "mtkv_get_total_cache_length", "mtkv_dump_page_map", "mtkv_state_blob", "mtkv_gen_config_default", "mtkv_gen_config_preset",
    "mtkv_generate_trace_jsonl", "mtkv_free", "mtkv_op_scatter_chunks", "mtkv_op_gather_chunks",
    "mtkv_op_paged_attention", "mtkv_op_paged_attention_batch", "mtkv_op_dense", "mtkv_attention_plan_check",
]

_lib = None


def lib():
    """Load libmtkv_b200.so (build it with ``python -m paper_2604_22881_b200.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise Error(f"{LIB_PATH} missing: run `python -m paper_2604_22881_b200.build` "
                    "(the serving path has no Python fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
    u32p = C.POINTER(C.c_uint32)
    sig = {
        "mtkv_last_error": (C.c_char_p, []),
        "mtkv_kv_config_default": (None, [C.POINTER(_KV)]),
        "mtkv_kv_config_validate": (C.c_int, [C.POINTER(_KV)]),
        "mtkv_parse_config_text": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(_KV)]),
        "mtkv_cost_model_default": (None, [C.POINTER(_Cost)]),
        "mtkv_pages_needed": (u64, [u64, u32]),
        "mtkv_persisted_prefix": (u64, [u64, u32]),
        "mtkv_planner_create": (vp, [C.POINTER(_KV), C.POINTER(_Cost), C.c_int]),
        "mtkv_planner_destroy": (None, [vp]),
        "mtkv_planner_process_batch": (C.c_int, [vp, C.POINTER(_Request), u32]),
        "mtkv_planner_drain": (C.c_int, [vp]),
        "mtkv_planner_set_onload_policy": (C.c_int, [vp, C.c_uint32, C.c_double, C.c_double]),
        "mtkv_engine_create": (vp, [C.POINTER(_KV), C.POINTER(_Cost), C.POINTER(_EngineOpts)]),
        "mtkv_engine_destroy": (None, [vp]),
        "mtkv_engine_process_batch": (C.c_int, [vp, C.POINTER(_Request), u32]),
        "mtkv_engine_run": (C.c_int, [vp, C.POINTER(_Request), u64, C.POINTER(_Report)]),
        "mtkv_engine_drain": (C.c_int, [vp]),
        "mtkv_engine_synchronize": (C.c_int, [vp]),
        "mtkv_engine_last_logits": (C.c_int, [vp, C.POINTER(C.c_float), u32]),
        "mtkv_engine_last_rankings": (C.c_int, [vp, u32p, u64]),
        "mtkv_engine_batch_rankings": (C.c_int, [vp, u64, u32p, u64]),
        "mtkv_engine_batches_submitted": (u64, [vp]),
        "mtkv_engine_last_plan_ms": (None, [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "mtkv_engine_check_conservation": (C.c_int, [vp]),
        "mtkv_engine_read_user_kv": (C.c_int64, [vp, u32, u32, C.POINTER(C.c_uint16),
                                                 C.POINTER(C.c_uint16), u64]),
        "mtkv_engine_last_batch_ms": (C.c_double, [vp]),
        "mtkv_engine_last_attention_ms": (C.c_double, [vp, u32p]),
        "mtkv_engine_last_proj_ms": (C.c_double, [vp, u32p, C.POINTER(C.c_uint64)]),
        "mtkv_engine_last_chunk_copy_ms": (C.c_int, [vp, C.POINTER(C.c_double), u32p, C.POINTER(C.c_double), u32p]),
        "mtkv_engine_kernel_launches": (u64, [vp]),
        "mtkv_engine_set_profile": (None, [vp, u32]),
        "mtkv_engine_set_onload_policy": (C.c_int, [vp, u32, C.c_double, C.c_double]),
        "mtkv_report": (C.c_int, [vp, C.c_int, C.POINTER(_Report)]),
        "mtkv_last_plans": (u32, [vp, C.c_int, C.POINTER(_Plan), u32]),
        "mtkv_last_evictions": (u32, [vp, C.c_int, C.POINTER(_Eviction), u32]),
        "mtkv_known_users": (u32, [vp, C.c_int, u32p, u32]),
        "mtkv_user_state": (C.c_int, [vp, C.c_int, u32, C.POINTER(_SeqState)]),
        "mtkv_user_pages": (u32, [vp, C.c_int, u32, u32p, u32]),
        "mtkv_lru_snapshot": (u32, [vp, C.c_int, u32p, u32]),
        "mtkv_evict_user": (C.c_int, [vp, C.c_int, u32]),
        "mtkv_is_locked": (C.c_int, [vp, C.c_int, u32]),
        "mtkv_get_total_cache_length": (u64, [vp, C.c_int, u32]),
        "mtkv_dump_page_map": (vp, [vp, C.c_int]),
        "mtkv_state_blob": (C.c_int64, [vp, C.c_int, C.POINTER(C.c_uint8), u64]),
        "mtkv_gen_config_default": (None, [C.POINTER(_GenCfg)]),
        "mtkv_gen_config_preset": (C.c_int, [C.c_char_p, C.POINTER(_GenCfg)]),
        "mtkv_generate_trace_jsonl": (vp, [C.POINTER(_GenCfg)]),
        "mtkv_free": (None, [vp]),
        "mtkv_op_scatter_chunks": (C.c_int, [vp, vp, vp, u32, C.POINTER(_KV), u32, vp]),
        "mtkv_op_gather_chunks": (C.c_int, [vp, vp, vp, u32, C.POINTER(_KV), u32, vp]),
        "mtkv_op_dense": (C.c_int, [vp, vp, vp, u32, u32, u32, u64, C.c_int, C.c_int, vp]),
        "mtkv_op_paged_attention": (C.c_int, [vp, vp, vp, vp, u32, u64, u64, u32, C.POINTER(_KV),
                                              u32, vp]),
        "mtkv_attention_plan_check": (C.c_int, [u32, u32p, u32p, C.POINTER(C.c_uint64), u32, u32, u32, u32, C.c_int,
                                                u32p]),
        "mtkv_op_paged_attention_batch": (C.c_int, [vp, vp, vp, vp, u32p, u32p, C.POINTER(C.c_uint64), u32, u32,
                                                    C.POINTER(_KV), u32, u32, C.POINTER(C.c_float), vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _err() -> str:
    return lib().mtkv_last_error().decode()


def _check(rc: int):
    if rc == 0:
        return
    msg = _err()
    if rc == 2:
        raise BatchRejected(msg)
    if rc == 3:
        raise NoDevice(msg)
    raise Error(msg)


# ------------------------------------------------------------ configuration ---
@dataclass
class KVConfig:
    """core.hpp:29 KVConfig (defaults: 8-layer HSTU serving config)."""
    num_layers: int = 8
    num_heads: int = 4
    head_dim: int = 128
    page_size: int = 32
    chunk_size: int = 1024
    device_pages: int = 40960
    onload_pages: int = 10008
    bytes_per_element: int = 2
    offload_quota: int = 8192
    host_capacity: int = 0

    def hidden(self) -> int:
        return self.num_heads * self.head_dim

    def pages_per_chunk(self) -> int:
        return self.chunk_size // self.page_size

    def token_kv_bytes(self) -> int:
        return self.num_layers * 2 * self.num_heads * self.head_dim * self.bytes_per_element

    def chunk_bytes(self) -> int:
        """bytes of one host chunk / staging slot: [L][2][chunk_size][H*D]"""
        return self.chunk_size * self.token_kv_bytes()

    def validate(self) -> None:
        _check(lib().mtkv_kv_config_validate(C.byref(self._c())))

    def _c(self) -> _KV:
        return _KV(**asdict(self))


@dataclass
class CostModel:
    """costs.hpp:11 CostModel — calibration of the deterministic event schedule."""
    bus_bandwidth: float = 25e9
    tx_setup: float = 10e-6
    host_bandwidth: float = 50e9
    page_op: float = 50e-9
    attn_coeff: float = 2e-10
    linear_coeff: float = 1e-7
    embed_coeff: float = 5e-8
    layout_coeff: float = 5e-8
    meta_fixed: float = 1e-4
    strip_fixed: float = 5e-5
    embed_fixed: float = 1e-4
    layout_fixed: float = 1e-4
    await_fixed: float = 5e-5
    update_fixed: float = 5e-5
    commit_per_chunk: float = 5e-6
    offload_submit: float = 3e-5
    post_fixed: float = 2e-4

    def _c(self) -> _Cost:
        return _Cost(**asdict(self))


@dataclass
class ModelConfig:
    """model.hpp:12 ModelConfig."""
    num_layers: int = 2
    num_heads: int = 2
    head_dim: int = 8
    vocab: int = 64
    seed: int = 1

    def hidden(self) -> int:
        return self.num_heads * self.head_dim


def parse_config_text(text: str, origin: str = "inline") -> KVConfig:
    """core.cpp:28 parse_config_text (key=value lines, '#' comments)."""
    out = _KV()
    _check(lib().mtkv_parse_config_text(text.encode(), origin.encode(), C.byref(out)))
    return KVConfig(**{f: getattr(out, f) for f, _ in _KV._fields_})


def load_config(path: str) -> KVConfig:
    """core.cpp:67 load_config."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise Error(f"config: cannot open {path}")
    return parse_config_text(text, path)


def pages_needed(length: int, page_size: int) -> int:
    if page_size < 1:
        raise Error("pages_needed: page size must be >= 1")
    return int(lib().mtkv_pages_needed(length, page_size))


def persisted_prefix(length: int, chunk_size: int) -> int:
    if chunk_size < 1:
        raise Error("persisted_prefix: chunk size must be >= 1")
    return int(lib().mtkv_persisted_prefix(length, chunk_size))


# ---------------------------------------------------------------- requests ---
class RequestBatch:
    """Packs requests (dicts in the reference JSONL schema: ts, user, dn, nc,
    optional tokens/cands) into the C struct array without per-token Python work."""

    def __init__(self, reqs: Sequence[dict]):
        n = len(reqs)
        self.n = n
        self.arr = (_Request * max(n, 1))()
        self._keep = []
        for i, r in enumerate(reqs):
            q = self.arr[i]
            q.timestamp = int(r.get("ts", 0))
            q.user = int(r["user"])
            toks, cands = r.get("tokens"), r.get("cands")
            if toks is not None and len(toks):
                a = np.ascontiguousarray(toks, dtype=np.uint32)
                self._keep.append(a)
                q.new_tokens = a.ctypes.data_as(C.POINTER(C.c_uint32))
                q.new_token_count = len(a)
            else:
                q.new_token_count = int(r.get("dn", 0)) if toks is None else 0
            if cands is not None and len(cands):
                b = np.ascontiguousarray(cands, dtype=np.uint32)
                self._keep.append(b)
                q.candidates = b.ctypes.data_as(C.POINTER(C.c_uint32))
                q.candidate_count = len(b)
            else:
                q.candidate_count = int(r.get("nc", 1))

    def candidate_counts(self) -> list[int]:
        return [self.arr[i].candidate_count for i in range(self.n)]


def batchify(trace: Sequence[dict], batch_size: int):
    """workload.cpp:247 batchify."""
    if batch_size < 1:
        raise Error("batchify: batch size must be >= 1")
    return [list(trace[i:i + batch_size]) for i in range(0, len(trace), batch_size)]


# ------------------------------------------------------------------ reports ---
def _report_dict(r: _Report) -> dict:
    d = {f: getattr(r, f) for f, _ in _Report._fields_ if f != "step_ms"}
    d["steps_ms"] = dict(zip(STEP_LABELS, list(r.step_ms)))
    return d


class _ManagerView:
    """Shared manager accessors (sim.hpp:149 manager()) for Planner and Engine."""
    _is_engine = 0

    def report(self) -> dict:
        r = _Report()
        _check(lib().mtkv_report(self._h, self._is_engine, C.byref(r)))
        return _report_dict(r)

    def plans(self) -> list[dict]:
        n = lib().mtkv_last_plans(self._h, self._is_engine, None, 0)
        arr = (_Plan * max(n, 1))()
        lib().mtkv_last_plans(self._h, self._is_engine, arr, n)
        return [{f: getattr(arr[i], f) for f, _ in _Plan._fields_} for i in range(n)]

    def evictions(self) -> list[dict]:
        n = lib().mtkv_last_evictions(self._h, self._is_engine, None, 0)
        arr = (_Eviction * max(n, 1))()
        lib().mtkv_last_evictions(self._h, self._is_engine, arr, n)
        return [{f: getattr(arr[i], f) for f, _ in _Eviction._fields_} for i in range(n)]

    def known_users(self) -> list[int]:
        n = lib().mtkv_known_users(self._h, self._is_engine, None, 0)
        a = (C.c_uint32 * max(n, 1))()
        lib().mtkv_known_users(self._h, self._is_engine, a, n)
        return list(a)[:n]

    def user_state(self, user: int) -> dict:
        s = _SeqState()
        _check(lib().mtkv_user_state(self._h, self._is_engine, user, C.byref(s)))
        return {f: getattr(s, f) for f, _ in _SeqState._fields_}

    def user_pages(self, user: int) -> list[int]:
        n = lib().mtkv_user_pages(self._h, self._is_engine, user, None, 0)
        a = (C.c_uint32 * max(n, 1))()
        lib().mtkv_user_pages(self._h, self._is_engine, user, a, n)
        return list(a)[:n]

    def lru_snapshot(self) -> list[int]:
        n = lib().mtkv_lru_snapshot(self._h, self._is_engine, None, 0)
        a = (C.c_uint32 * max(n, 1))()
        lib().mtkv_lru_snapshot(self._h, self._is_engine, a, n)
        return list(a)[:n]

    def evict_user(self, user: int) -> None:
        _check(lib().mtkv_evict_user(self._h, self._is_engine, user))

    def is_locked(self, user: int) -> bool:
        return bool(lib().mtkv_is_locked(self._h, self._is_engine, user))

    def get_total_cache_length(self, user: int) -> int:
        return int(lib().mtkv_get_total_cache_length(self._h, self._is_engine, user))

    def dump_page_map(self) -> str:
        """Engine<B>::dump_page_map (sim.hpp:493): same JSON text as the reference."""
        p = lib().mtkv_dump_page_map(self._h, self._is_engine)
        try:
            return C.string_at(p).decode()
        finally:
            lib().mtkv_free(p)

    def state_blob(self) -> bytes:
        """Canonical binary image of the control-plane state (mtkv_state_blob)."""
        n = lib().mtkv_state_blob(self._h, self._is_engine, None, 0)
        buf = (C.c_uint8 * n)()
        lib().mtkv_state_blob(self._h, self._is_engine, buf, n)
        return bytes(buf)

    def state(self) -> dict:
        """Full control-plane state, same schema as the reference driver's dump."""
        users = []
        for u in self.known_users():
            s = self.user_state(u)
            users.append(dict(user=u, total_len=s["total_len"], device_len=s["device_len"],
                              persisted_len=s["persisted_len"], locked=bool(s["locked"]),
                              last_access=s["last_access"], pages=self.user_pages(u),
                              host_chunks=s["host_chunks"], pending_offload=s["pending_offload"]))
        r = self.report()
        return dict(users=users, lru=self.lru_snapshot(), evictions=r["evictions"],
                    tail_tokens_lost=r["tail_tokens_lost"], pages_allocated=r["pages_allocated"],
                    occupied_pages=r["occupied_pages"], free_pages=r["free_pages"],
                    quota_in_flight=r["quota_in_flight"], clock=r["clock"])


class Planner(_ManagerView):
    """Host control plane (CacheManager + Pipeline schedule of Engine<B>), no payloads."""
    _is_engine = 0

    def __init__(self, kv: KVConfig, cost: CostModel | None = None, mode: str = "hierarchical"):
        self.kv = kv
        self._h = lib().mtkv_planner_create(C.byref(kv._c()), C.byref((cost or CostModel())._c()),
                                            MODE[mode])
        if not self._h:
            raise Error(_err())

    def __del__(self):
        if getattr(self, "_h", None):
            lib().mtkv_planner_destroy(self._h)
            self._h = None

    def process_batch(self, batch: Sequence[dict]) -> None:
        rb = RequestBatch(batch)
        _check(lib().mtkv_planner_process_batch(self._h, rb.arr, rb.n))

    def drain(self) -> None:
        _check(lib().mtkv_planner_drain(self._h))

    def set_onload_policy(self, policy: str, onload_gbs: float, recompute_mtok_s: float) -> None:
        """The executor's host-hit split as the planner applies it at fixed rates
        (report: prefix_recomputed / prefix_onloaded); decisions are unchanged."""
        if policy not in ("always", "adaptive"):
            raise Error(f"unknown onload policy {policy!r}")
        _check(lib().mtkv_planner_set_onload_policy(self._h, int(policy == "adaptive"), onload_gbs, recompute_mtok_s))


class Ticket:
    """Handle of a submitted batch (Engine.submit)."""
    __slots__ = ("batch", "counts")

    def __init__(self, batch: int, counts: list[int]):
        self.batch, self.counts = batch, counts


class Engine(_ManagerView):
    """sim.hpp:110 Engine<B> with the data plane on a B200 (sm_100a kernels)."""
    _is_engine = 1

    def __init__(self, kv: KVConfig, cost: CostModel | None = None, mode: str = "hierarchical",
                 backend: str = "tag", batch_size: int = 1, model: ModelConfig | None = None,
                 device: int = 0, keep_logits: bool = False, profile: bool = False, seed: int = 1,
                 host_reserve_mb: int = 0, planner: str = "host", max_users: int = 0,
                 max_user_pages: int = 0, host_extent_mb: int = 0, onload_policy: str = "always",
                 onload_gbs: float = 0.0, recompute_mtok_s: float = 0.0):
        self.kv, self.mode, self.backend, self.batch_size = kv, mode, backend, batch_size
        self.model = model
        if backend == "value" and model is None:
            raise Error("value backend requires model params")
        o = _EngineOpts()
        o.mode, o.backend, o.batch_size, o.seed = MODE[mode], BACKEND[backend], batch_size, seed
        if model is not None:
            o.model = _ModelCfg(model.num_layers, model.num_heads, model.head_dim, model.vocab, model.seed)
        o.device, o.keep_logits, o.profile = device, int(keep_logits), int(profile)
        o.host_reserve_mb = int(host_reserve_mb)
        if planner not in ("host", "device"):
            raise Error("planner must be 'host' or 'device'")
        o.device_planner = int(planner == "device")
        o.max_users, o.max_user_pages = int(max_users), int(max_user_pages)
        o.host_extent_mb = int(host_extent_mb)
        if onload_policy not in ("always", "adaptive"):
            raise Error("onload_policy must be 'always' or 'adaptive'")
        o.onload_policy = int(onload_policy == "adaptive")
        o.onload_gbs, o.recompute_mtok_s = float(onload_gbs), float(recompute_mtok_s)
        self._h = lib().mtkv_engine_create(C.byref(kv._c()), C.byref((cost or CostModel())._c()),
                                           C.byref(o))
        if not self._h:
            msg = _err()
            if "no CUDA device" in msg or "device ordinal" in msg:
                raise NoDevice(msg)
            raise Error(msg)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().mtkv_engine_destroy(self._h)
            self._h = None

    def process_batch(self, batch, packed: RequestBatch | None = None) -> None:
        rb = packed or RequestBatch(batch)
        _check(lib().mtkv_engine_process_batch(self._h, rb.arr, rb.n))

    def submit(self, batch=None, packed: RequestBatch | None = None) -> "Ticket":
        """Pipelined serving: enqueue a batch and return a ticket for its results
        (read them with rankings(ticket) while later batches are in flight)."""
        rb = packed or RequestBatch(batch)
        _check(lib().mtkv_engine_process_batch(self._h, rb.arr, rb.n))
        return Ticket(int(lib().mtkv_engine_batches_submitted(self._h)) - 1, rb.candidate_counts())

    def rankings(self, ticket: "Ticket") -> list[list[int]]:
        """rank_candidates (model.cpp:199) of every request of the ticket's batch."""
        tot = sum(ticket.counts)
        out = np.zeros(max(tot, 1), dtype=np.uint32)
        n = lib().mtkv_engine_batch_rankings(self._h, ticket.batch, out.ctypes.data_as(C.POINTER(C.c_uint32)), tot)
        if n < 0:
            raise Error(_err())
        res, o = [], 0
        for c in ticket.counts:
            res.append(out[o:o + c].tolist())
            o += c
        return res

    def run(self, trace: Sequence[dict]) -> dict:
        """sim.hpp:135 run(): batchify, process, drain, report."""
        for b in batchify(trace, self.batch_size):
            self.process_batch(b)
        self.drain()
        return self.report()

    def drain(self) -> None:
        _check(lib().mtkv_engine_drain(self._h))

    def synchronize(self) -> None:
        _check(lib().mtkv_engine_synchronize(self._h))

    def last_logits(self) -> np.ndarray:
        rows = len(self.plans())
        out = np.zeros((max(rows, 1), self.model.vocab), dtype=np.float32)
        n = lib().mtkv_engine_last_logits(self._h, out.ctypes.data_as(C.POINTER(C.c_float)), rows)
        if n < 0:
            raise Error(_err())
        return out[:n]

    def last_rankings(self) -> list[list[int]]:
        plans = self.plans()
        tot = sum(p["num_candidates"] for p in plans)
        out = np.zeros(max(tot, 1), dtype=np.uint32)
        n = lib().mtkv_engine_last_rankings(self._h, out.ctypes.data_as(C.POINTER(C.c_uint32)), tot)
        if n < 0:
            raise Error(_err())
        res, o = [], 0
        for p in plans:
            res.append(out[o:o + p["num_candidates"]].tolist())
            o += p["num_candidates"]
        return res

    def check_conservation(self) -> None:
        _check(lib().mtkv_engine_check_conservation(self._h))

    def read_user_kv(self, user: int, layer: int):
        """Resident K/V of one layer in logical order as raw bf16 bits [len x H*D]."""
        st = self.user_state(user)
        d = self.kv.hidden()
        n = st["device_len"]
        k = np.zeros((max(n, 1), d), dtype=np.uint16)
        v = np.zeros((max(n, 1), d), dtype=np.uint16)
        got = lib().mtkv_engine_read_user_kv(self._h, user, layer,
                                             k.ctypes.data_as(C.POINTER(C.c_uint16)),
                                             v.ctypes.data_as(C.POINTER(C.c_uint16)), n)
        if got < 0:
            raise Error(_err())
        return k[:got], v[:got]

    def last_batch_ms(self) -> float:
        return float(lib().mtkv_engine_last_batch_ms(self._h))

    def last_attention_ms(self):
        n = C.c_uint32(0)
        ms = lib().mtkv_engine_last_attention_ms(self._h, C.byref(n))
        return float(ms), int(n.value)

    def last_plan_ms(self):
        """(host planning wall ms, device planner kernel ms) of the last batch."""
        a, b = C.c_double(), C.c_double()
        lib().mtkv_engine_last_plan_ms(self._h, C.byref(a), C.byref(b))
        return a.value, b.value

    def last_proj_ms(self):
        """(ms, launches, rows) of the last batch's projection GEMMs (profile mode)."""
        n, rows = C.c_uint32(), C.c_uint64()
        ms = lib().mtkv_engine_last_proj_ms(self._h, C.byref(n), C.byref(rows))
        return float(ms), int(n.value), int(rows.value)

    def last_chunk_copy_ms(self):
        """(scatter_ms, scatter_chunks, gather_ms, gather_chunks) of the last batch (profile mode)."""
        sm, gm = C.c_double(), C.c_double()
        sc, gc = C.c_uint32(), C.c_uint32()
        _check(lib().mtkv_engine_last_chunk_copy_ms(self._h, C.byref(sm), C.byref(sc), C.byref(gm), C.byref(gc)))
        return sm.value, sc.value, gm.value, gc.value

    def set_profile(self, on: bool) -> None:
        lib().mtkv_engine_set_profile(self._h, int(on))

    def set_onload_policy(self, policy: str, onload_gbs: float = 0.0, recompute_mtok_s: float = 0.0) -> None:
        """'always' (every host hit onloaded, as the reference) or 'adaptive'
        (some host-hit prefixes re-encoded on the SMs); from the next batch on."""
        if policy not in ("always", "adaptive"):
            raise Error("onload_policy must be 'always' or 'adaptive'")
        _check(lib().mtkv_engine_set_onload_policy(self._h, int(policy == "adaptive"), onload_gbs, recompute_mtok_s))

    def kernel_launches(self) -> int:
        return int(lib().mtkv_engine_kernel_launches(self._h))


# ----------------------------------------------------------------- workload ---
@dataclass
class GenConfig:
    """workload.hpp:15 GenConfig."""
    num_users: int = 100
    total_requests: int = 2000
    pareto: bool = False
    gap_log_mu: float = 9.0
    gap_log_sigma: float = 1.5
    pareto_alpha: float = 1.3
    pareto_scale_ms: float = 1000.0
    mean_final_len: float = 6375.0
    min_len: int = 1
    max_len: int = 20000
    fixed_delta: int = 0
    candidates: int = 5
    vocab: int = 0
    seed: int = 42

    @staticmethod
    def preset(name: str) -> "GenConfig":
        g = _GenCfg()
        _check(lib().mtkv_gen_config_preset(name.encode(), C.byref(g)))
        return GenConfig(**{f: (bool(getattr(g, f)) if f == "pareto" else getattr(g, f))
                            for f, _ in _GenCfg._fields_})


def generate_trace(g: GenConfig) -> list[dict]:
    """workload.cpp:85 generate_trace — same RNG streams, same records."""
    c = _GenCfg(**{k: (int(v) if k == "pareto" else v) for k, v in asdict(g).items()})
    p = lib().mtkv_generate_trace_jsonl(C.byref(c))
    if not p:
        raise Error(_err())
    text = C.string_at(p).decode()
    lib().mtkv_free(p)
    return [json.loads(x) for x in text.splitlines() if x]


def rank_candidates(logits, candidates) -> list[int]:
    """model.cpp:199 rank_candidates: stable descending sort by logit."""
    for c in candidates:
        if c >= len(logits):
            raise Error("rank_candidates: candidate id out of range")
    return sorted(candidates, key=lambda c: -float(logits[c]))


def attention_cost(total: int, cached: int) -> int:
    """model.hpp:72 attention_cost."""
    if cached > total:
        raise Error("attention_cost: cached prefix exceeds total")
    return (total - cached) * total
