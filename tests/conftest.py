import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libshellular_cuda.so")
    config.addinivalue_line("markers", "slow: long-running CPU oracle cases")


@pytest.fixture(scope="session")
def S():
    import paper_2511_04025_b200 as S
    return S


@pytest.fixture(scope="session")
def O():
    import oracle as O
    return O


@pytest.fixture(scope="session")
def ctx(S):
    return S.default_context(0)
