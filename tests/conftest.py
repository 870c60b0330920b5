import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a kernels")
    config.addinivalue_line("markers", "slow: long-running case")
    # Build the native library and the CPU checkers when absent (e.g. a fresh
    # GPU box that received sources only); a no-op when up to date.
    from paper_2011_01805_b200 import build
    build.build_product()
    build.build_oracle()


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import load_oracle
    return load_oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_lib import load_ref
    r = load_ref()
    if r is None:
        pytest.skip("reference library oracle/_ref not built here (no /root/reference)")
    return r


def _has_gpu() -> bool:
    try:
        from paper_2011_01805_b200 import device_count
        return device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not _has_gpu():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return True


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
