import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the fused CUDA kernels)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.pyoracle import REF_SO, Reference

    if not os.path.exists(REF_SO) and not os.path.isdir("/root/reference/proj/core"):
        pytest.skip("reference library not built and sources absent")
    return Reference()


@pytest.fixture(scope="session")
def native():
    import paper_1209_2137_b200 as P

    P._native.lib()
    return P


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    return torch
