"""GPU parity at every BASELINE.json config shape on REFERENCE-encoded
buffers (tests/config_cases.py): C1 ClusterData d=29, C2 b = 0..32 raw, C3
d in {18,22,26,29} x {cluster, uniform} x {D1, D4}, C4 at 1/5/10% outliers,
a C5 sample (both codecs).  Every decode path is held to the reference's
decode_array / decode_deltas word for word: the fused kernels (izg_decode),
the workspace path (izg_decode_ws: page index + indexed decode, or the split
kernel for small batches), the host-buffer path (izg_decode_host), and —
in fresh processes, since the switches are read once — the one-warp
indexed path (IZG_SPLIT=0 IZG_TEAM=0), the split kernel everywhere (IZG_SPLIT=1), the
large-batch indexed shape (IZG_BIG_IDX_BATCH=1) and the SIMD-BP128 group
kernels (IZG_GROUP=2/8) and the lane-per-page index pass
(IZG_INDEX_LANES_MIN=0), each with the CTA kernel off (IZG_CTA=0; it is the
default for these small SIMD-BP128 batches and is forced onto the same
cases by tests/test_gpu_cta.py).  The team SIMD-FastPFOR kernel (the default
from 128 pages on) is forced onto the same cases by tests/test_gpu_team.py."""
import os
import subprocess
import sys

import pytest

from tests import config_cases as CC

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cases(ref):
    return CC.all_cases(ref)


def test_default_paths(cuda, cases):
    labels = {c["label"].split()[0] for c in cases}
    assert labels == {"C1", "C2", "C3", "C4", "C5"}
    CC.check_gpu(cases)


@pytest.mark.parametrize("env", [{"IZG_SPLIT": "0", "IZG_CTA": "0", "IZG_TEAM": "0"},
                                 {"IZG_SPLIT": "1", "IZG_CTA": "0"},
                                 {"IZG_SPLIT": "0", "IZG_BIG_IDX_BATCH": "1", "IZG_CTA": "0",
                                  "IZG_TEAM": "0"},
                                 {"IZG_SPLIT": "0", "IZG_GROUP": "2", "IZG_CTA": "0"},
                                 {"IZG_SPLIT": "0", "IZG_GROUP": "8", "IZG_CTA": "0"},
                                 {"IZG_SPLIT": "0", "IZG_INDEX_LANES_MIN": "0", "IZG_TEAM": "0"}],
                         ids=["one-warp", "split", "big-idx", "group2", "group8", "lane-index"])
def test_forced_paths(cuda, ref, env):
    r = subprocess.run([sys.executable, "-m", "tests.config_cases"], cwd=ROOT,
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]
