"""C-ABI boundary: the library loads, exports every symbol include/*.h declares,
and its host-side entry points keep the reference's semantics (no GPU needed)."""
import glob
import hashlib
import json
import os
import re

import pytest

import paper_2604_22881_b200 as mtkv
from tests.util import ROOT, golden


def _declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        for m in re.finditer(r"\b(mtkv_[a-z0-9_]+)\s*\(", text):
            names.add(m.group(1))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    lib = mtkv.lib()
    declared = _declared_symbols()
    assert len(declared) >= 40
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(mtkv.EXPORTED_SYMBOLS)


def test_page_and_chunk_geometry():
    """test_core.cpp:7."""
    assert mtkv.pages_needed(0, 32) == 0
    assert mtkv.pages_needed(1, 32) == 1
    assert mtkv.pages_needed(32, 32) == 1
    assert mtkv.pages_needed(33, 32) == 2
    assert mtkv.pages_needed(320064, 32) == 10002
    assert mtkv.persisted_prefix(0, 1024) == 0
    assert mtkv.persisted_prefix(1023, 1024) == 0
    assert mtkv.persisted_prefix(1024, 1024) == 1024
    assert mtkv.persisted_prefix(5189, 1024) == 5120
    with pytest.raises(mtkv.Error):
        mtkv.pages_needed(10, 0)


def test_config_defaults_validation_and_parsing():
    """test_core.cpp:23-64."""
    c = mtkv.KVConfig()
    assert c.hidden() == 512 and c.pages_per_chunk() == 32 and c.token_kv_bytes() == 16384
    c.validate()
    for bad in (dict(chunk_size=48), dict(offload_quota=100), dict(page_size=0)):
        with pytest.raises(mtkv.Error):
            mtkv.KVConfig(**bad).validate()
    cfg = mtkv.parse_config_text("# comment\npage_size = 16\nchunk_size = 64   # inline\n\ndevice_pages=128\n")
    assert (cfg.page_size, cfg.chunk_size, cfg.device_pages, cfg.num_layers) == (16, 64, 128, 8)
    with pytest.raises(mtkv.Error, match="x:1: unknown key 'nope'"):
        mtkv.parse_config_text("nope = 3\n", "x")
    with pytest.raises(mtkv.Error):
        mtkv.parse_config_text("page_size\n", "x")
    with pytest.raises(mtkv.Error):
        mtkv.parse_config_text("page_size = abc\n", "x")
    with pytest.raises(mtkv.Error):
        mtkv.load_config("/nonexistent/path.cfg")


def test_generator_reproduces_reference_traces():
    """The product generator draws the reference's RNG streams (workload.cpp:85)."""
    for case in golden("traces"):
        g = dict(case["gen"])
        base = mtkv.GenConfig.preset(g.pop("preset")) if "preset" in g else mtkv.GenConfig()
        for k, v in g.items():
            setattr(base, k, v)
        t = mtkv.generate_trace(base)
        assert len(t) == case["n"]
        assert t[:5] == case["head"]
        assert hashlib.sha256(json.dumps(t, sort_keys=True).encode()).hexdigest() == case["digest"]


def test_generator_validation_and_presets():
    """test_workload.cpp:515."""
    assert mtkv.GenConfig.preset("kuairand1k").num_users == 1000
    assert mtkv.GenConfig.preset("mt").min_len == 4000
    with pytest.raises(mtkv.Error):
        mtkv.GenConfig.preset("imaginary")
    with pytest.raises(mtkv.Error):
        mtkv.generate_trace(mtkv.GenConfig(mean_final_len=1e9))
    with pytest.raises(mtkv.Error):
        mtkv.generate_trace(mtkv.GenConfig(total_requests=0))


def test_rank_candidates_and_attention_cost():
    """test_model.cpp:236 / :243."""
    assert mtkv.rank_candidates([0.0, 5.0, 5.0, -1.0], [3, 2, 1, 0]) == [2, 1, 0, 3]
    with pytest.raises(mtkv.Error):
        mtkv.rank_candidates([0.0], [7])
    assert mtkv.attention_cost(10, 0) == 100 and mtkv.attention_cost(10, 10) == 0
    with pytest.raises(mtkv.Error):
        mtkv.attention_cost(5, 6)


def test_engine_without_gpu_fails_loudly():
    """No CPU fallback: on a machine without a CUDA device the engine refuses."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(mtkv.NoDevice):
        mtkv.Engine(mtkv.KVConfig(num_layers=1, num_heads=1, head_dim=8, device_pages=8))
