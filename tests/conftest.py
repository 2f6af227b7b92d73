import os
import sys

import pytest

# The oracle's OpenMP loops must not busy-wait at their barriers: on a loaded host (other
# jobs on the cores) spinning threads starve each other and a test of tiny problems slows by
# orders of magnitude.  Set before the oracle library is loaded.
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: full-size case (minutes)")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")
