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


def gpu_shared_by_processes() -> bool:
    """True when several processes may hold contexts on GPU 0 at once (compute
    mode DEFAULT): the multi-process tests need it (IPC peers, torchrun ranks
    sharing the one GPU of the box)."""
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        return pynvml.nvmlDeviceGetComputeMode(h) == pynvml.NVML_COMPUTEMODE_DEFAULT
    except Exception:
        return True  # cannot tell: try


needs_shared_gpu = pytest.mark.skipif(not gpu_shared_by_processes(),
                                      reason="GPU 0 is not in DEFAULT compute mode (one process per GPU)")
