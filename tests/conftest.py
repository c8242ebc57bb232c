import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference, compiled in place (oracle/_ref/libarf_ref.so)."""
    from oracle.oracle_ctypes import REF_LIB, Checker, build
    if not REF_LIB.exists():
        if Path("/root/reference/proj/include/arf").is_dir():
            build("ref")
        else:
            pytest.skip("oracle/_ref/libarf_ref.so not built and /root/reference absent")
    return Checker("ref")


@pytest.fixture(scope="session")
def oracle():
    """Our C restatement (oracle/_build/libarf_oracle.so), built on demand."""
    from oracle.oracle_ctypes import ORACLE_LIB, Checker, build
    if not ORACLE_LIB.exists():
        build("oracle")
    return Checker("oracle")


@pytest.fixture(scope="session")
def gpu():
    from paper_2212_10550_b200 import arf
    from paper_2212_10550_b200._lib import LIB_PATH
    if not LIB_PATH.exists():
        from paper_2212_10550_b200.build import build
        build()
    n = arf.device_count()
    if n == 0:
        pytest.fail("GPU test selected but no CUDA device is visible")
    return arf
