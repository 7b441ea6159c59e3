"""Consumer of the decoded arrays: GPU intersection of two
decoded posting lists against numpy.intersect1d of the original arrays (the
oracle: intersect1d's sorted-unique semantics; the reference has no
intersection API).  Edge cases: empty, disjoint, identical, repeated values,
one list much shorter than the other, values at 0 and 2^32-1, tile edges."""
import numpy as np
import pytest
import torch

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
    got = P.intersect(codec, P.encode_array(codec, a), P.encode_array(codec, b))
    assert np.array_equal(got, np.intersect1d(a, b))
