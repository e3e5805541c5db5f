"""The C++ drop-in (include/mtkv_b200_engine.hpp) under the reference's own test
cases: tests/cpp/test_dropin.cpp runs each case against the unmodified
reference and against the B200 path and requires identical observable results
(see its header for the case list and file:line citations). The binary is built
by `make -C oracle dropin` (part of __graft_entry__.build() wherever the
reference sources are present) and travels with the snapshot."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_dropin")

needs_bin = pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/test_dropin not built "
                               "(make -C oracle dropin needs /root/reference)")


@needs_bin
def test_dropin_manager_cases_match_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@needs_bin
@pytest.mark.gpu
def test_dropin_engine_and_manager_cases_match_reference_on_gpu():
    r = subprocess.run([BIN, "--engine"], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "sim: value backend logits are mode-invariant" in r.stdout and "0 failed" in r.stdout
