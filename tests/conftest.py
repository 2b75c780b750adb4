import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle, build

    build(ref=False)
    return Oracle("oracle")


@pytest.fixture(scope="session")
def ref():
    from oracle import Oracle

    if not Oracle.available("ref"):
        from oracle import build

        try:
            build(ref=True)
        except Exception:  # pragma: no cover - reference absent on this machine
            pass
    if not Oracle.available("ref"):
        pytest.skip("oracle/_ref/libpbsref.so not built (reference absent here)")
    return Oracle("ref")


GOLDEN = os.path.join(ROOT, "tests", "golden")
