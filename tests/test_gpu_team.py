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


_HEAVY = r'''
import sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import paper_1209_2137_b200 as P
from oracle.pyoracle import Oracle
from tests.page_builder import build_fastpfor_page
O = Oracle()
rng = np.random.default_rng(5)

def blocks(n, kind):
    out = []
    for k in range(n):
        low = rng.integers(0, 2**32, size=128, dtype=np.uint64)
        if kind == "overflow":      # 255 exceptions per block, one width: cursors pass 65,535,
            b, mb, c = 7, 19, 255   # 8 KiB of position bytes per 32 blocks
        elif kind == "widths":      # 100 exceptions per block, widths 1..32 in turn: most
            b, mb, c = 0, 1 + k % 32, 100   # super-iterations need two groups per width (17.9 KB
                                            # of packed groups, over a window), some one (9.5 KB)
        elif kind == "windows":     # several windows per page, all staged
            b = int(rng.integers(0, 12)); mb = b + int(rng.integers(1, 21)); c = int(rng.integers(20, 60))
        else:                       # sparse
            b = int(rng.integers(0, 33)); mb = min(32, b + int(rng.integers(0, 3))); c = int(rng.integers(1, 4)) if mb > b else 0
        pos = [int(x) for x in rng.integers(0, 128, size=c)]
        if kind != "overflow":
            pos = sorted(pos)
        highs = [int(x) for x in rng.integers(0, 2**32, size=c, dtype=np.uint64)]
        out.append((low, b, mb, pos, highs))
    return out

def d4(x):
    y = x.astype(np.uint64).reshape(-1, 4).cumsum(axis=0) & 0xFFFFFFFF
    return y.reshape(-1).astype(np.uint32)

pages, expects = [], []
for kind, n in [("overflow", 512), ("widths", 512), ("windows", 512), ("sparse", 512),
                ("windows", 70), ("widths", 33), ("overflow", 1), ("sparse", 97)] * 20:
    page, expect = build_fastpfor_page(blocks(n, kind), True)
    pages.append(page); expects.append(expect)
flat = np.concatenate(expects)
for name in ("simdfastpfor", "simdfastpfor-s4"):
    codec = P.make_codec(name)
    enc = P.layout(codec, pages, [len(e) for e in expects])
    assert len(pages) >= 128  # the team kernel's default range too
    b = P.DeviceBatch(codec, enc, raw=True)
    b.decode()
    assert not b.statuses().any()
    assert np.array_equal(b.output(), flat)
    assert list(b.consumed[:b.n_chunks].cpu().numpy()) == [len(p) for p in pages]
    a = P.DeviceBatch(codec, enc)   # array mode: the prefix sum on top
    a.decode()
    assert not a.statuses().any()
    want = np.concatenate([d4(e) if name.endswith("s4") else (np.cumsum(e.astype(np.uint64)) & 0xFFFFFFFF).astype(np.uint32) for e in expects])
    assert np.array_equal(a.output(), want)
# a position >= 128 late in a heavy page: same status as the oracle and the fused kernel
bad = [p.copy() for p in pages[:8]]
for p in bad:
    A = int(p[0]); L = int(p[A])
    ba = p[A + 1: A + 1 + (L + 3) // 4].view(np.uint8)
    s = 0; last = None
    while s < L:
        bb, mb = int(ba[s]), int(ba[s + 1])
        if mb > bb:
            last = s + 3 + int(ba[s + 2]) - 1
            s += 3 + int(ba[s + 2])
        else:
            s += 2
    ba[last] = 200
codec = P.make_codec("simdfastpfor")
enc = P.layout(codec, bad, [len(e) for e in expects[:8]])
team = P.DeviceBatch(codec, enc, raw=True); team.decode()
fused = P.DeviceBatch(codec, enc, raw=True, indexed=False); fused.decode()
st = [O.decode_deltas("simdfastpfor", p, len(e))[0] for p, e in zip(bad, expects[:8])]
assert list(team.statuses()) == list(fused.statuses()) == st and all(st), (team.statuses(), st)
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


@pytest.mark.parametrize("lanes", ["0", "1000000000"], ids=["lane-index", "warp-index"])
def test_team_kernel_heavy_pages(cuda, lanes):
    """Pages that leave the team kernel's staged paths: cursors past 65,535
    and 8 KiB of position bytes per super-iteration (patch from global
    memory), a super-iteration whose packed exception groups exceed a
    window, many windows per page, short pages; raw and array mode, and the
    position-range status on a corrupted heavy page."""
    _run({"IZG_TEAM": "1", "IZG_SPLIT": "0", "IZG_INDEX_LANES_MIN": lanes},
         _HEAVY.format(root=ROOT))


@pytest.mark.parametrize("lanes", ["0", "1000000000"], ids=["lane-index", "warp-index"])
def test_team_kernel_random_batches(cuda, lanes):
    """tools/team_stress.py for 15 s: random batch sizes, ragged lengths with
    VByte remainders, data models, outlier rates and delta modes, every batch
    decoded three times and compared with the generated arrays word for word
    (a 10-minute run of the same tool covered 835,000 arrays)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "team_stress.py"), "15", "7"],
                       cwd=ROOT, env=dict(os.environ, IZG_TEAM="1", IZG_INDEX_LANES_MIN=lanes),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().startswith("ok"), r.stdout[-1000:] + r.stderr[-3000:]


def test_team_kernel_config_shapes(cuda, ref):
    _run({"IZG_TEAM": "1", "IZG_SPLIT": "0"},
         f"import sys; sys.path.insert(0, {ROOT!r}); from tests.config_cases import main; main()")
