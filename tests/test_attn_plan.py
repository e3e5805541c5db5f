"""Attention work planner (attn_plan.cpp), host-only: every (request, head,
query tile, key tile) is assigned to exactly one persistent CTA, CTAs get
balanced tile counts, partial slots are contiguous per segment."""
import numpy as np
import pytest

import paper_2604_22881_b200 as mtkv


def _check(n_hist, n_cand, start, H=2, D=128, S=32, ctas=148, tc=1):
    n = len(n_hist)
    a = lambda x, t: np.ascontiguousarray(x, dtype=t)
    nh, nc, st = a(n_hist, np.uint32), a(n_cand, np.uint32), a(start, np.uint64)
    stats = np.zeros(5, dtype=np.uint32)
    u32p = lambda x: x.ctypes.data_as(mtkv.C.POINTER(mtkv.C.c_uint32))
    rc = mtkv.lib().mtkv_attention_plan_check(n, u32p(nh), u32p(nc), st.ctypes.data_as(mtkv.C.POINTER(mtkv.C.c_uint64)),
                                              H, D, S, ctas, tc, u32p(stats))
    assert rc == 0, f"plan check failed with code {rc}"
    return stats


@pytest.mark.parametrize("seed", range(6))
def test_plan_covers_every_tile_once(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 80))
    n_hist = rng.integers(0, 300, n)
    n_cand = rng.integers(1, 9, n)
    start = rng.integers(0, 9000, n)
    for H, S, ctas in ((2, 32, 148), (4, 16, 148), (1, 64, 7), (3, 8, 148)):
        segs, pieces, tiles, max_cta, nctas = (int(x) for x in _check(n_hist, n_cand, start, H=H, S=S, ctas=ctas))
        assert nctas <= ctas and max_cta * nctas >= tiles
        assert max_cta <= 2 * -(-tiles // nctas) + 1  # balanced ranges (head lists are equal length)


def test_plan_bench_batch_balanced():
    """The bench layer: 64 requests, ~4.2 K keys, 72..199 fresh rows."""
    rng = np.random.default_rng(0)
    n = 64
    tail = np.where(rng.random(n) < 0.69, rng.integers(0, 128, n), 0)
    segs, pieces, tiles, max_cta, nctas = (int(x) for x in _check(64 + tail, np.full(n, 8),
                                                                   4096 + 64 * rng.integers(0, 16, n)))
    assert nctas == 148
    assert max_cta <= tiles / nctas * 1.05 + 1


def test_plan_mma_path_items():
    _check([5, 100, 0], [1, 3, 8], [0, 500, 7], H=2, D=32, S=8, tc=0)


@pytest.mark.parametrize("seed", range(6))
def test_paired_plan_covers_every_tile_once(seed):
    """Paired query tiles (attn_pair_kernel): every tile of both segments of a
    unit is covered exactly once, the B slot belongs to the next query tile of
    the same (request, head), and A only takes the key tiles it can see."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 40))
    # prefill-shaped (many query tiles) mixed with decode-shaped requests
    n_hist = np.where(rng.random(n) < 0.5, rng.integers(129, 4200, n), rng.integers(0, 200, n))
    n_cand = rng.integers(1, 9, n)
    start = np.where(rng.random(n) < 0.5, 0, rng.integers(0, 9000, n))
    for H, S, ctas in ((2, 32, 148), (1, 64, 7), (4, 16, 148)):
        segs, pieces, tiles, max_cta, nctas = (int(x) for x in _check(n_hist, n_cand, start, H=H, S=S, ctas=ctas, tc=2))
        assert nctas <= ctas and max_cta * nctas >= tiles
        assert max_cta <= 2 * -(-tiles // nctas) + 1


def test_paired_plan_halves_key_tiles_of_a_prefill():
    """A 4 K causal prefill: pairing streams each key tile once per two query tiles."""
    single = _check([4096] * 8, [8] * 8, [0] * 8, tc=1)
    paired = _check([4096] * 8, [8] * 8, [0] * 8, tc=2)
    assert paired[2] < 0.56 * single[2]
