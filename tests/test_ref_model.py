"""Pins the torch fp64 restatement (tests/ref_model.py) to the reference: the
reference's forward_incremental outputs (tests/golden/forward.json, generated
by the unmodified reference) and the C oracle's fp64 forward."""
import numpy as np

from oracle.oracle import ModelParams
from tests.ref_model import RefModel, RefServer
from tests.util import golden


def test_ref_model_matches_reference_forward_goldens():
    for case in golden("forward"):
        p = ModelParams(**case["model"])
        m = RefModel(p)
        split = case["split"]
        hist, cands = case["history"], case["candidates"]
        ck = cv = None
        if split:
            _, k, v = m.forward(None, None, hist[:split], [0])
            ck, cv = [x[:split] for x in k], [x[:split] for x in v]
        logits, _, _ = m.forward(ck, cv, hist[split:], cands)
        ref = np.array(case["logits"])
        got = logits.numpy()
        assert np.abs(got - ref).max() <= 1e-9 * max(np.abs(ref).max(), 1e-300), case["model"]


def test_ref_server_incremental_equals_full_forward():
    """Serving a user's history in several requests gives the full forward's
    logits (causal attention: the incremental path is exact)."""
    p = ModelParams(num_layers=2, num_heads=2, head_dim=8, vocab=50, seed=3)
    m = RefModel(p)
    rng = np.random.default_rng(0)
    toks = rng.integers(0, 50, 90).tolist()
    cands = [3, 7]
    srv = RefServer(m)
    for a, b in [(0, 40), (40, 41), (41, 75)]:
        srv.serve(1, toks[a:b], cands)
    inc = srv.serve(1, toks[75:], cands).numpy()
    full, _, _ = m.forward(None, None, toks, cands)
    full = full.numpy()
    assert np.abs(inc - full).max() <= 1e-10 * np.abs(full).max()
    c_logits, _, _ = p.forward(toks, cands)
    assert np.abs(full - c_logits).max() <= 1e-9 * np.abs(c_logits).max()
