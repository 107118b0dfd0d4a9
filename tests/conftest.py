import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def pytest_sessionstart(session):
    # the oracle is test infrastructure: build it if missing (gcc only)
    lib = ROOT / "oracle" / "_build" / "liboracle.so"
    if not lib.exists():
        import subprocess
        subprocess.run(["make", "-C", str(ROOT / "oracle")], check=True, capture_output=True)


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2509_26222_b200 import terrain
    return terrain.Context.default(0)
