"""Seeded input generators (bench/test harness): determinism and the
properties each BASELINE.json recipe promises."""
import numpy as np
import pytest

import harness as H
import paper_1209_2137_b200 as P


@pytest.mark.parametrize("model,d", [("uniform", 18), ("uniform", 29), ("cluster", 20),
                                     ("cluster", 29)])
def test_sorted_distinct_in_range(native, model, d):
    v, dd = H.gen_arrays(model, 8, 65536, d, seed=11, threads=2)
    assert np.all(dd == d)
    for row in v:
        assert np.all(np.diff(row.astype(np.int64)) > 0)
        assert int(row.max()) < (1 << d)


def test_deterministic_and_seeded_per_array(native):
    a, _ = H.gen_arrays("cluster", 6, 4096, (20, 29), seed=5, threads=3)
    b, _ = H.gen_arrays("cluster", 6, 4096, (20, 29), seed=5, threads=1)
    assert np.array_equal(a, b)
    c, _ = H.gen_arrays("cluster", 3, 4096, (20, 29), seed=8, threads=1)
    assert np.array_equal(a[3:], c)  # array i uses seed + i (datagen.cpp:129-134)


def test_per_array_width_range(native):
    _, d = H.gen_arrays("cluster", 2000, 256, (20, 29), seed=1, threads=4)
    assert d.min() == 20 and d.max() == 29
    counts = np.bincount(d, minlength=30)[20:]
    assert counts.min() > 120  # roughly uniform over the 10 widths


def test_cluster_is_clustered(native):
    """ClusterData concentrates values: its D4 deltas compress better than
    uniform at the same density (the point of the model)."""
    cu, _ = H.gen_arrays("uniform", 16, 65536, 29, seed=2)
    cc, _ = H.gen_arrays("cluster", 16, 65536, 29, seed=2)
    codec = P.make_codec("simdbp128-s4")
    bits = []
    for v in (cu, cc):
        e = H.encode_chunks(codec, v.reshape(-1), np.arange(16, dtype=np.uint64) * 65536,
                            np.full(16, 65536, np.uint32))
        bits.append(32 * e.payload_words / v.size)
    assert bits[1] < bits[0] - 1.0


def test_geometric_outliers(native):
    v, _ = H.gen_arrays("geometric", 4, 65536, 32, seed=3, rate_ppm=100000)
    gaps = np.diff(v.astype(np.uint64), axis=1) % (1 << 32)
    big = gaps >= 4096
    assert 0.08 < big.mean() < 0.12
    small = gaps[~big]
    assert 7.0 < small.mean() < 9.5  # geometric mean 8 (outlier draws excluded)
    assert small.min() >= 1


def test_raw_width(native):
    for b in (0, 1, 7, 31, 32):
        v, _ = H.gen_arrays("raw", 2, 4096, b, seed=4)
        assert int(v.max()) < (1 << b) if b < 32 else True
        if b:
            assert int(v.max()) >= (1 << (b - 1))
