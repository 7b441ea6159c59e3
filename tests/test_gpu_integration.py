"""INTEGRATION.md's C++ binding, compiled (oracle/Makefile) against the
reference's headers and library: intzip::decode_array_b200 must equal
intzip::decode_array — same output, and on corrupted chunks the same
exception type and what() (tests/cpp/test_integration.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_integration")


def _binary():
    if not os.path.exists(BIN):
        pytest.skip("integration binary not built (reference sources absent at build time)")
    return BIN


@pytest.mark.gpu
def test_decode_array_b200_equals_reference(cuda):
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " 0 failures" in r.stdout


def test_binding_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=300)
    # every GPU decode raises (no CPU fallback): the comparison fails
    assert r.returncode != 0 and "b200 decode failed" in r.stdout
