import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the checker (oracle) and the product library if they are missing."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "_build", "libmtkv_oracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    if not os.path.exists(os.path.join(ROOT, "paper_2604_22881_b200", "libmtkv_b200.so")):
        subprocess.run([sys.executable, "-m", "paper_2604_22881_b200.build"], check=True, cwd=ROOT)
    yield
