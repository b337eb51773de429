import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    oracle.port()
    return oracle


@pytest.fixture(scope="session")
def tp():
    import paper_2510_27351_b200 as tp

    return tp
