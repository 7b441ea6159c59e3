"""The team SIMD-FastPFOR decode (csrc/team.cuh: one CTA of 8 warps per page,
shared TMA staging of packed words / block records / position bytes,
windowed bulk unpack of the exception arrays into shared memory, two-level
prefix sum) forced onto the parity suites (IZG_TEAM=1, read once per
process, hence subprocesses): outputs, statuses and words consumed against
the oracle, the reference and the fused path — edge lengths, VByte
remainders, unaligned placements, mutation fuzz, structural mutations of
every page field, duplicate / c = 255 / w = 32 exception cases, and the
BASELINE config shapes encoded by the reference — behind both page index
passes (warp per page, lane per page)."""
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
from tests import test_gpu_indexed as TI
from tests import test_collisions as TC
O, R = Oracle(), Reference()
for name in ["simdfastpfor", "simdfastpfor-s4", "simdfastpfor-d2", "simdfastpfor-dm"]:
    T.test_roundtrip_assorted(torch, O, name)
    for wp, op in [(1, 0), (2, 3), (0, 2), (3, 1)]:
        T.test_unaligned_placement(torch, name, wp, op)
    T.test_mutation_fuzz_matches_oracle(torch, O, name)
for name in ["simdfastpfor", "simdfastpfor-s4"]:
    T.test_reference_encoded_buffers_decode(torch, R, name)
    T.test_mutation_fuzz_accept_reject_matches_reference(torch, R, name)
    T.test_decode_deltas_every_width(torch, R, name)
    TI.test_structural_mutations_raw(torch, O, name)
T.test_device_checksum_large_batch(torch, "simdfastpfor-s4")
for name in TI.FP_NAMES:
    TI.test_structural_mutations_array(torch, O, name)
    TI.test_random_byte_fuzz_both_paths(torch, name)
TC.test_collisions_on_gpu(torch, O, True)
print("ok")
'''


def _run(env, code, timeout=1200):
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), \
        r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("lanes", ["0", "1000000000"], ids=["lane-index", "warp-index"])
def test_team_kernel_parity_suite(cuda, lanes):
    _run({"IZG_TEAM": "1", "IZG_SPLIT": "0", "IZG_INDEX_LANES_MIN": lanes},
         _SCRIPT.format(root=ROOT))


def test_team_kernel_config_shapes(cuda, ref):
    _run({"IZG_TEAM": "1", "IZG_SPLIT": "0"},
         f"import sys; sys.path.insert(0, {ROOT!r}); from tests.config_cases import main; main()")
