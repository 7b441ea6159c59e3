import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _ensure_built():
    """Fresh checkouts carry no binaries: build the library (nvcc) and the
    parity checkers (gcc/g++) once, in-tree, before the first test."""
    lib = os.path.join(ROOT, "paper_1209_2137_b200", "_lib", "libintzip_b200.so")
    orc = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
    ref = os.path.join(ROOT, "oracle", "_ref", "libintzip_ref.so")
    hz = os.path.join(ROOT, "harness", "_build", "libizh.so")
    need_ref = not os.path.exists(ref) and os.path.isdir("/root/reference/proj/core")
    if not os.path.exists(lib) or not os.path.exists(orc) or not os.path.exists(hz) or need_ref:
        import __graft_entry__

        __graft_entry__.build()


def pytest_configure(config):
    _ensure_built()
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
