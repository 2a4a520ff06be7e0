import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")
    # build the oracle (and oracle/_ref when the reference tree is present)
    # before collection, so skipif(not have_ref()) reflects this container and
    # never skips a reference-pinning test only because the build came later
    from oracle import oracle as O
    O.build()


@pytest.fixture(scope="session")
def built():
    """Compile the oracle (and oracle/_ref when the reference tree exists) and the engine."""
    from oracle import oracle as O
    O.build()
    from paper_1612_00595_b200 import build as B
    B.build()
    return True
