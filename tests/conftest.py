import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libgsim_gpu.so")
    config.addinivalue_line("markers", "slow: full-size parity cases")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Ref, REF_LIB
    if not REF_LIB.exists() and not Path("/root/reference/proj").exists():
        pytest.skip("reference library oracle/_ref not built here")
    return Ref()


@pytest.fixture(scope="session")
def ctx():
    """A CUDA context on device 0. Fails (does not skip) when the library cannot run: the
    gpu tests are the parity gate and must never pass on a fallback."""
    from paper_2507_21981_b200 import Context
    return Context(0)
