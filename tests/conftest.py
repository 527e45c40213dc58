import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); parity tests through the C ABI")


@pytest.fixture(scope="session")
def co():
    """The plain-C oracle (always available: built from oracle/tw_oracle.c)."""
    from oracle.py import COracle
    return COracle()


@pytest.fixture(scope="session")
def ref():
    """The compiled, unmodified reference (oracle/_ref), when present."""
    from oracle.py import RefOracle, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefOracle()


@pytest.fixture(scope="session")
def ref_philox():
    from oracle.py import RefOracle, ref_available
    if not ref_available(philox=True):
        pytest.skip("oracle/_ref philox build absent")
    return RefOracle(philox=True)


@pytest.fixture(scope="session")
def tw():
    """The product package (GPU). Fails loudly if the library is missing."""
    import paper_2605_16182_b200 as tw
    return tw
