"""Split decode (csrc/split.cuh: several warps per chunk, decoupled look-back
carry) against the one-warp-per-chunk kernel and the original arrays.

Small batches take the split kernel whenever a workspace is given
(DeviceBatch(indexed=True)); DeviceBatch(indexed=False) runs izg_decode, the
one-warp kernel, which the parity suites pin to the reference.  Small
SIMD-BP128 array batches now default to the CTA kernel (csrc/cta.cuh) on
both sides, so the SIMD-BP128 split paths are exercised in subprocesses with
IZG_CTA=0 (test_split_large_batch_forced, test_split_segment_sizes).  Outputs must
match word for word and statuses exactly, including under corruption (the
first error of a chunk in stream order travels with the look-back)."""
import numpy as np
import pytest

import harness as H
import paper_1209_2137_b200 as P
from paper_1209_2137_b200 import _native as N
from paper_1209_2137_b200.codec import Encoded
from tests.helpers import random_sorted

pytestmark = pytest.mark.gpu

ARRAY_NAMES = ["simdbp128", "simdbp128-s4", "simdbp128-d2", "simdbp128-dm", "simdfastpfor",
               "simdfastpfor-s4", "simdfastpfor-d2", "simdfastpfor-dm"]
LENGTHS = [1, 3, 127, 128, 129, 2047, 2048, 2049, 4095, 4096, 4097, 8192, 30000, 61441,
           65535, 65536]


def batch_of(codec, arrays, allow_wrap=False):
    flat = np.concatenate(arrays).astype(np.uint32)
    counts = np.array([len(a) for a in arrays], np.uint32)
    offs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64)
    return flat, H.encode_chunks(codec, flat, offs, counts, allow_wrap=allow_wrap)


def both(codec, enc, raw=False):
    split = P.DeviceBatch(codec, enc, raw=raw)
    one = P.DeviceBatch(codec, enc, raw=raw, indexed=False)
    assert split.workspace is not None  # small batch: the split kernel runs
    split.decode()
    one.decode()
    return split, one


def test_workspace_selects_split(cuda):
    L = N.lib()
    assert L.izg_decode_workspace_size(0, 100) > 0  # SIMD-BP128: look-back state
    assert L.izg_decode_workspace_size(1, 100) > 100 * (16 + 128 + 512 * 16)
    assert L.izg_decode_workspace_size(0, 1 << 16) == 0  # large batches: one warp per chunk


@pytest.mark.parametrize("name", ARRAY_NAMES)
def test_split_arrays(cuda, name):
    codec = P.make_codec(name)
    rng = np.random.default_rng(abs(hash(name)) % 1000)
    arrays = [random_sorted(rng, n, int(rng.integers(1, 5000))) for n in LENGTHS]
    flat, enc = batch_of(codec, arrays)
    s, o = both(codec, enc)
    s.check()
    o.check()
    assert np.array_equal(s.output(), flat)
    assert np.array_equal(o.output(), flat)
    assert np.array_equal(s.consumed[:s.n_chunks].cpu().numpy(),
                          o.consumed[:o.n_chunks].cpu().numpy())


@pytest.mark.parametrize("name", ["simdfastpfor-s4", "simdfastpfor", "simdbp128-s4"])
def test_split_outliers(cuda, name):
    """C4-like pages: many exceptions, wrapping sums, every segment patched."""
    codec = P.make_codec(name)
    vals, _ = H.gen_arrays("geometric", 6, 65536, 32, seed=5, rate_ppm=100000)
    arrays = [v for v in vals] + [vals[0][:40000]]
    flat, enc = batch_of(codec, arrays, allow_wrap=True)
    s, o = both(codec, enc)
    s.check()
    assert np.array_equal(s.output(), flat)
    assert np.array_equal(s.output(), o.output())


def test_split_multichunk_array(cuda):
    """One long array (chunks of 2^16 and a ragged tail chunk) in one batch."""
    codec = P.make_codec("simdbp128-s4")
    rng = np.random.default_rng(1)
    flat = random_sorted(rng, 5 * 65536 + 777, 60)
    enc = H.encode_array(codec, flat)
    s, o = both(codec, enc)
    s.check()
    assert np.array_equal(s.output(), flat)


@pytest.mark.parametrize("name", ["simdbp128", "simdfastpfor"])
def test_split_raw(cuda, name):
    """Codec-level decode_deltas (no delta coding): counts multiple of 128."""
    codec = P.make_codec(name)
    rng = np.random.default_rng(2)
    counts = np.array([128, 4096, 65536, 8192 + 128, 640], np.uint32)
    vals = (rng.integers(0, 1 << 32, int(counts.sum()), dtype=np.uint64)
            >> rng.integers(0, 32, int(counts.sum()), dtype=np.uint64)).astype(np.uint32)
    offs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64)
    enc = H.encode_chunks(codec, vals, offs, counts, raw=True)
    s, o = both(codec, enc, raw=True)
    s.check()
    assert np.array_equal(s.output(), vals)
    assert np.array_equal(s.consumed[:s.n_chunks].cpu().numpy(),
                          o.consumed[:o.n_chunks].cpu().numpy())


@pytest.mark.parametrize("name", ["simdbp128-s4", "simdfastpfor-s4", "simdbp128", "simdfastpfor"])
def test_split_corruption_statuses(cuda, name):
    """Random word corruptions in multi-segment chunks: the split path reports
    exactly the one-warp path's status per chunk (first error in stream
    order), and identical output for chunks that still decode."""
    codec = P.make_codec(name)
    rng = np.random.default_rng(11)
    arrays = [random_sorted(rng, 65536, 40) for _ in range(4)] + [random_sorted(rng, 30001, 9)]
    _, enc = batch_of(codec, arrays)
    for trial in range(40):
        w = enc.words.copy()
        for _ in range(int(rng.integers(1, 4))):
            c = int(rng.integers(0, len(enc.table)))
            off = int(enc.table["word_off"][c])
            nw = int(enc.table["n_words"][c])
            i = off + int(rng.integers(0, nw))
            w[i] ^= np.uint32(1) << np.uint32(rng.integers(0, 32))
        bad = Encoded(w, enc.table)
        s, o = both(codec, bad)
        st_s, st_o = s.statuses(), o.statuses()
        assert np.array_equal(st_s, st_o), (trial, st_s, st_o)
        ok = np.nonzero(st_o == 0)[0]
        so, oo = s.output(), o.output()
        for c in ok:
            a = int(enc.table["out_off"][c])
            n = int(enc.table["n"][c])
            assert np.array_equal(so[a:a + n], oo[a:a + n]), (trial, c)


_LARGE = r'''
import sys
sys.path.insert(0, {root!r})
import harness as H
import numpy as np, paper_1209_2137_b200 as P
for name, model, d, rate, count in [("simdbp128-s4", "cluster", 29, 0, 2048),
                                    ("simdfastpfor-s4", "geometric", 32, 100000, 1024)]:
    codec = P.make_codec(name)
    vals, _ = H.gen_arrays(model, count, 65536, d, seed=1, rate_ppm=rate)
    enc = H.encode_chunks(codec, vals.reshape(-1), np.arange(count, dtype=np.uint64) * 65536,
                          np.full(count, 65536, np.uint32), allow_wrap=model == "geometric")
    b = P.DeviceBatch(codec, enc)
    for rep in range(3):
        b.out.fill_(0)
        b.decode()
        b.check()
        bad = int((b.output().reshape(count, 65536) != vals).any(axis=1).sum())
        assert bad == 0, (name, rep, bad)
print("ok")
'''


def test_split_large_batch_forced():
    """Thousands of chunks through the split kernel (IZG_SPLIT=1), so warps
    run many units each and predecessors publish while successors poll: the
    regime in which a partly published prefix once leaked into a carry."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, IZG_SPLIT="1", IZG_CTA="0")
    r = subprocess.run([sys.executable, "-c", _LARGE.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


_SEGS = r'''
import sys
sys.path.insert(0, {root!r})
import torch
from tests import test_gpu_split as T
for name in ["simdbp128", "simdbp128-s4", "simdbp128-dm", "simdbp128-d2"]:
    T.test_split_arrays(torch, name)
for name in ["simdbp128-s4", "simdbp128"]:
    T.test_split_corruption_statuses(torch, name)
print("ok")
'''


@pytest.mark.parametrize("segs", [1, 2, 4, 8])
def test_split_segment_sizes(segs):
    """SIMD-BP128 sizes its segments to the batch (split_seg_blocks): every
    size, forced with IZG_SPLIT_SEGS, against the one-warp kernel — outputs,
    words consumed, and statuses under corruption (each unit walks the
    descriptor chain from the chunk start; an error on an earlier segment is
    reported by its own unit)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, IZG_SPLIT_SEGS=str(segs), IZG_CTA="0")
    r = subprocess.run([sys.executable, "-c", _SEGS.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]
