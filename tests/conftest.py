import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a kernels)")


@pytest.fixture(scope="session")
def corc():
    """The plain-C oracle restatement (built on demand)."""
    from oracle.oracle import COracle

    return COracle()


@pytest.fixture(scope="session")
def rorc():
    """The unmodified reference build (oracle/_ref); skipped where it was not built."""
    from oracle.oracle import REF_LIB, RefOracle

    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref not built (reference headers absent)")
    return RefOracle()


@pytest.fixture(scope="session")
def orc():
    """Best checker available: the reference build, else the C restatement."""
    from oracle.oracle import best_available

    return best_available()


@pytest.fixture(scope="session")
def P():
    import paper_1202_1060_b200

    return paper_1202_1060_b200
