import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long CPU oracle runs")


@pytest.fixture(scope="session")
def restated():
    from oracle.pyoracle import Restated

    return Restated()


@pytest.fixture(scope="session")
def reference():
    from oracle.pyoracle import Reference, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def gpu():
    from paper_2405_08764_b200.engine import device_count

    if device_count() < 1:
        pytest.fail("GPU test selected but no CUDA device is visible")
    return True


def rel_err(a, b):
    import numpy as np

    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))
