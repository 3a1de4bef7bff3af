"""Test configuration: `gpu` marks tests that need a B200 (run with -m gpu)."""
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 device (B200)")


@pytest.fixture(scope="session")
def lib():
    from paper_2408_13510_b200 import abi, build
    build.build()
    return abi.load_library()


@pytest.fixture(scope="session")
def gpu(lib):
    """The engine on a real device; fails (never skips) when none is usable."""
    n = lib.rs_device_count()
    if n < 1:
        pytest.fail("no sm_100 device visible: GPU tests must run on a B200")
    return lib
