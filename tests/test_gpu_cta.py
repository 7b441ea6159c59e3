"""The CTA-cooperative SIMD-BP128 kernel (csrc/cta.cuh: one CTA per SM, a
shared staging ring filled by a producer warp, units of 1,024 integers round
robin over 16 consumer warps with a mailbox carry) forced onto the parity
suites (IZG_CTA=1, read once per process, hence subprocesses): outputs and
statuses against the oracle and the reference on every array mode, edge
lengths, VByte remainders, unaligned placements, mutation fuzz, and the
BASELINE config shapes encoded by the reference."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r'''
import sys
sys.path.insert(0, {root!r})
import torch
from oracle.pyoracle import Oracle, Reference
from tests import test_gpu_parity as T
O, R = Oracle(), Reference()
for name in ["simdbp128", "simdbp128-s4", "simdbp128-d2", "simdbp128-dm"]:
    T.test_roundtrip_assorted(torch, O, name)
    for wp, op in [(1, 0), (2, 3), (0, 2)]:
        T.test_unaligned_placement(torch, name, wp, op)
    T.test_mutation_fuzz_matches_oracle(torch, O, name)
for name in ["simdbp128", "simdbp128-s4"]:
    T.test_reference_encoded_buffers_decode(torch, R, name)
    T.test_mutation_fuzz_accept_reject_matches_reference(torch, R, name)
T.test_device_checksum_large_batch(torch, "simdbp128-s4")
print("ok")
'''


def _run(env, code, timeout=900):
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), \
        r.stdout[-2000:] + r.stderr[-4000:]


def test_cta_kernel_parity_suite(cuda):
    _run({"IZG_CTA": "1", "IZG_SPLIT": "0"}, _SCRIPT.format(root=ROOT))


def test_cta_kernel_config_shapes(cuda, ref):
    _run({"IZG_CTA": "1", "IZG_SPLIT": "0"},
         f"import sys; sys.path.insert(0, {ROOT!r}); from tests.config_cases import main; main()")
