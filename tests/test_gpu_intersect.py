"""Consumer of the decoded arrays: GPU intersection of two
decoded posting lists against numpy.intersect1d of the original arrays (the
oracle: intersect1d's sorted-unique semantics; the reference has no
intersection API).  Edge cases: empty, disjoint, identical, repeated values,
one list much shorter than the other, values at 0 and 2^32-1, tile edges."""
import numpy as np
import pytest
import torch

import harness as H
import paper_1209_2137_b200 as P
from tests.helpers import random_sorted

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).cuda()


def check(a, b):
    got = P.intersect_device(dev(a), dev(b)).cpu().numpy().view(np.uint32)
    want = np.intersect1d(a, b)
    assert np.array_equal(got, want), (len(a), len(b), len(got), len(want))


def test_edges(cuda):
    z = np.zeros(0, np.uint32)
    check(z, z)
    check(z, np.arange(10, dtype=np.uint32))
    check(np.arange(10, dtype=np.uint32), z)
    check(np.arange(5000, dtype=np.uint32), np.arange(5000, 9000, dtype=np.uint32))  # disjoint
    check(np.arange(0, 3000, 2, dtype=np.uint32), np.arange(1, 3000, 2, dtype=np.uint32))
    x = np.arange(0, 1 << 20, 3, dtype=np.uint32)
    check(x, x)
    check(np.array([0, 0, 0, 5, 5, 0xFFFFFFFF, 0xFFFFFFFF], np.uint32),
          np.array([0, 5, 5, 5, 7, 0xFFFFFFFF], np.uint32))
    for n in (1023, 1024, 1025, 2047, 2048, 4097):  # tile edges (1024 per tile)
        a = np.arange(n, dtype=np.uint32) * 2
        check(a, np.arange(3 * n, dtype=np.uint32))


@pytest.mark.parametrize("na,nb", [(100, 10 ** 6), (10 ** 5, 10 ** 5), (3 * 10 ** 6, 50_000)])
def test_random_lists(cuda, na, nb):
    rng = np.random.default_rng(na + nb)
    a = random_sorted(rng, na, 40)
    b = random_sorted(rng, nb, 40 * max(1, na // nb)) if nb < na else random_sorted(rng, nb, 7)
    check(a, b)


@pytest.mark.parametrize("name", ["simdbp128-s4", "simdfastpfor-s4", "simdbp128"])
def test_decode_then_intersect(cuda, name):
    """The composed query: both lists decoded on the GPU, intersected there,
    only the common values copied back."""
    rng = np.random.default_rng(9)
    codec = P.make_codec(name)
    a = random_sorted(rng, 200_000, 60)
    b = np.unique(np.concatenate([a[rng.random(len(a)) < 0.3],
                                  random_sorted(rng, 150_000, 80)])).astype(np.uint32)
    got = P.intersect(codec, H.encode_array(codec, a), H.encode_array(codec, b))
    assert np.array_equal(got, np.intersect1d(a, b))


# ---- fused decode -> intersect (izg_decode_intersect) ---------------------

ALL_NAMES = ["simdbp128-s4", "simdbp128", "simdfastpfor-s4", "simdfastpfor", "bp32",
             "bp32-s4", "fastpfor", "fastpfor-s4", "simplepfor", "simplepfor-s4"]


def encode_any(name, flat):
    codec = P.make_codec(name)
    if codec.codec in (0, 1):
        return codec, H.encode_array(codec, flat)
    from oracle.pyoracle import Reference

    ch = Reference().encode_array(name, flat)
    return codec, P.layout(codec, [p for _, p in ch], [n for n, _ in ch])


def fused(name, long_, s):
    codec, enc = encode_any(name, long_)
    b = P.DeviceBatch(codec, enc, materialize=False, indexed=False)
    got = P.decode_intersect_device(b, dev(s)).cpu().numpy().view(np.uint32)
    b.check()
    return got


@pytest.mark.parametrize("name", ALL_NAMES)
def test_fused_codecs(cuda, name):
    """Every codec, ragged lengths (VByte tails), several chunks, a probe list
    holding repeats and values outside the decoded range."""
    rng = np.random.default_rng(17)
    long_ = random_sorted(rng, 140_000, 90)  # 3 chunks, 8,928-integer tail chunk
    s = np.sort(np.concatenate([long_[rng.random(len(long_)) < 0.05],
                                rng.integers(0, 1 << 24, 5000, dtype=np.uint32),
                                long_[:3], long_[-3:], [0, 0xFFFFFFFF]]).astype(np.uint32))
    assert np.array_equal(fused(name, long_, s), np.intersect1d(long_, s))


@pytest.mark.parametrize("n", [1, 5, 127, 128, 129, 2047, 2049, 65535, 65536, 65537])
def test_fused_lengths(cuda, n):
    rng = np.random.default_rng(n)
    long_ = random_sorted(rng, n, 9)
    s = np.unique(np.concatenate([long_[::3], long_ + 1])).astype(np.uint32)
    for name in ("simdbp128-s4", "simdfastpfor-s4"):
        assert np.array_equal(fused(name, long_, s), np.intersect1d(long_, s)), name


def test_fused_edges(cuda):
    rng = np.random.default_rng(3)
    long_ = random_sorted(rng, 70_000, 50)
    z = np.zeros(0, np.uint32)
    assert len(fused("simdbp128-s4", long_, z)) == 0
    # probe list longer than the decoded list, dense: many rounds per tile
    s = np.arange(0, int(long_[-1]) + 100, dtype=np.uint32)
    assert np.array_equal(fused("simdfastpfor-s4", long_, s), np.unique(long_))
    # runs of equal values in both lists, straddling tiles (every value x 700)
    long_ = np.repeat(np.arange(200, dtype=np.uint32) * 7, 700)
    s = np.repeat(np.arange(300, dtype=np.uint32) * 3, 3)
    assert np.array_equal(fused("simdbp128-s4", long_, s), np.intersect1d(long_, s))
    # long runs of repeats in the probe list straddling hit words and
    # 1,024-element compaction groups
    long_ = random_sorted(np.random.default_rng(4), 50_000, 5)
    s = np.repeat(np.unique(np.concatenate([long_[::7], long_[::11] + 1])), 37).astype(np.uint32)
    assert np.array_equal(fused("simdbp128-s4", long_, s), np.intersect1d(long_, s))
    # values at the top of the range
    long_ = (np.uint32(0xFFFFFFFF) - np.arange(1000, dtype=np.uint32)[::-1])
    s = np.array([0, 0xFFFFFFF0, 0xFFFFFFFE, 0xFFFFFFFF], np.uint32)
    assert np.array_equal(fused("simdbp128", long_, s), np.intersect1d(long_, s))
    # disjoint
    assert len(fused("simdfastpfor-s4", np.arange(1000, dtype=np.uint32) * 2,
                     np.arange(1000, dtype=np.uint32) * 2 + 1)) == 0


def test_fused_several_arrays(cuda):
    """Chunks of several arrays in one call: the decoded values form one set."""
    rng = np.random.default_rng(5)
    arrs = [random_sorted(rng, int(rng.integers(1, 30_000)), 30) for _ in range(12)]
    codec = P.make_codec("simdfastpfor-s4")
    flat = np.concatenate(arrs)
    counts = np.array([len(a) for a in arrs], np.uint32)
    offs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64)
    enc = H.encode_chunks(codec, flat, offs, counts)
    s = np.unique(rng.integers(0, int(flat.max()) + 1, 20_000, dtype=np.uint32))
    b = P.DeviceBatch(codec, enc, materialize=False, indexed=False)
    got = P.decode_intersect_device(b, dev(s)).cpu().numpy().view(np.uint32)
    b.check()
    assert np.array_equal(got, np.intersect1d(flat, s))


def test_fused_status(cuda):
    """A corrupt chunk reports the same status as izg_decode."""
    rng = np.random.default_rng(8)
    long_ = random_sorted(rng, 65536 * 2, 40)
    codec = P.make_codec("simdbp128-s4")
    enc = H.encode_array(codec, long_)
    w = enc.words.copy()
    w[int(enc.table["word_off"][1])] = 0xFFFFFFFF  # widths > 32 in chunk 1
    from paper_1209_2137_b200.codec import Encoded

    bad = Encoded(w, enc.table)
    b = P.DeviceBatch(codec, bad, materialize=False, indexed=False)
    P.decode_intersect_device(b, dev(long_[:100]))
    ref = P.DeviceBatch(codec, bad)
    ref.decode()
    st, st_ref = b.statuses(), ref.statuses()
    assert st[0] == 0 and st[1] != 0
    assert np.array_equal(st, st_ref)


@pytest.mark.parametrize("name", ["simdbp128-s4", "simdfastpfor-s4"])
def test_intersect_fused_matches_unfused(cuda, name):
    rng = np.random.default_rng(21)
    codec = P.make_codec(name)
    a = random_sorted(rng, 300_000, 40)
    b = np.unique(np.concatenate([a[rng.random(len(a)) < 0.1],
                                  random_sorted(rng, 20_000, 600)])).astype(np.uint32)
    ea, eb = H.encode_array(codec, a), H.encode_array(codec, b)
    want = np.intersect1d(a, b)
    assert np.array_equal(P.intersect(codec, ea, eb, fused=True), want)
    assert np.array_equal(P.intersect(codec, ea, eb, fused=False), want)
