"""GPU encoder (secondary path): words identical to the reference encoder's,
and GPU-encoded buffers decode on the CPU reference and on the GPU."""
import zlib

import numpy as np
import pytest

import harness as H
import paper_1209_2137_b200 as P
from paper_1209_2137_b200.device import encode_on_device
from tests.helpers import assorted_arrays, chunks_of, random_sorted

pytestmark = pytest.mark.gpu

BP_NAMES = ["simdbp128", "simdbp128-s4", "simdbp128-d2", "simdbp128-dm"]
FP_NAMES = ["simdfastpfor", "simdfastpfor-s4", "simdfastpfor-d2", "simdfastpfor-dm"]


def _chunks(arr):
    offs = np.arange(0, len(arr), 65536, dtype=np.uint64)
    counts = np.minimum(65536, len(arr) - offs).astype(np.uint32)
    return offs, counts


@pytest.mark.parametrize("name", BP_NAMES + FP_NAMES)
def test_gpu_encode_matches_host_encoder(cuda, name):
    codec = P.make_codec(name)
    for arr in assorted_arrays(seed=zlib.crc32(name.encode()) % 101):
        offs, counts = _chunks(arr)
        genc, st = encode_on_device(codec, arr, offs, counts)
        assert np.all(st == 0)
        henc = H.encode_chunks(codec, arr, offs, counts)
        for (n1, a), (n2, b) in zip(chunks_of(genc), chunks_of(henc)):
            assert n1 == n2 and np.array_equal(a, b), (name, len(arr))
        assert np.array_equal(P.decode_array(codec, genc), arr)


@pytest.mark.parametrize("name", ["simdbp128", "simdbp128-s4", "simdfastpfor", "simdfastpfor-s4"])
def test_gpu_encode_matches_reference(cuda, ref, name):
    codec = P.make_codec(name)
    rng = np.random.default_rng(8)
    for n in (1, 5, 129, 2048, 2049 + 64, 65536, 65536 + 300):
        arr = random_sorted(rng, n, int(rng.choice([3, 1000, 1 << 20])))
        offs, counts = _chunks(arr)
        genc, st = encode_on_device(codec, arr, offs, counts)
        assert np.all(st == 0)
        theirs = ref.encode_array(name, arr)
        for (n1, a), (n2, b) in zip(chunks_of(genc), theirs):
            assert n1 == n2 and np.array_equal(a, b)


@pytest.mark.parametrize("codec_name", ["simdbp128", "simdfastpfor"])
def test_gpu_encode_raw_every_width(cuda, ref, codec_name):
    codec = P.make_codec(codec_name)
    rng = np.random.default_rng(9)
    vals, counts = [], []
    for b in range(33):
        n = 128 * (1 + b % 20)
        v = (rng.integers(0, 2**32, size=n, dtype=np.uint64) & ((1 << b) - 1)).astype(np.uint32)
        if b % 3 == 0:  # outliers: FastPFOR exceptions of many widths
            v[::29] = rng.integers(0, 2**32, size=len(v[::29]), dtype=np.uint64)
        vals.append(v)
        counts.append(n)
    flat = np.concatenate(vals)
    offs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64)
    genc, st = encode_on_device(codec, flat, offs, counts, raw=True)
    assert np.all(st == 0)
    for (n, w), v in zip(chunks_of(genc), vals):
        assert np.array_equal(w, ref.encode_deltas(codec_name, v))


@pytest.mark.parametrize("name", ["simdbp128-s4", "simdfastpfor-s4"])
def test_gpu_encode_wrap_and_decreasing(cuda, ref, name):
    codec = P.make_codec(name)
    vals, _ = H.gen_arrays("geometric", 3, 65536, 32, seed=4, rate_ppm=50000)
    flat = vals.reshape(-1)
    offs, counts = np.arange(3, dtype=np.uint64) * 65536, np.full(3, 65536, np.uint32)
    _, st = encode_on_device(codec, flat, offs, counts)
    assert np.all(st == 66)  # delta.cpp:13 (sums wrap, so D4 sees a decrease)
    genc, st = encode_on_device(codec, flat, offs, counts, allow_wrap=True)
    assert np.all(st == 0)
    for i, (n, w) in enumerate(chunks_of(genc)):
        assert np.array_equal(w, ref.encode_chunk_wrapping(name, vals[i]))
    bad = np.array([5, 3] + list(range(10, 300)), np.uint32)
    _, st = encode_on_device(P.make_codec("simdbp128"), bad, np.array([0], np.uint64),
                             np.array([len(bad)], np.uint32))
    assert st[0] == 66


@pytest.mark.parametrize("name", ["simdbp128-s4", "simdfastpfor-s4"])
def test_gpu_encode_large_batch_roundtrip(cuda, name):
    codec = P.make_codec(name)
    vals, _ = H.gen_arrays("cluster", 512, 65536, (20, 29), seed=77)
    flat = vals.reshape(-1)
    offs, counts = np.arange(512, dtype=np.uint64) * 65536, np.full(512, 65536, np.uint32)
    genc, st = encode_on_device(codec, flat, offs, counts)
    assert np.all(st == 0)
    henc = H.encode_chunks(codec, flat, offs, counts)
    assert genc.payload_words == henc.payload_words
    b = P.DeviceBatch(codec, genc)
    b.decode()
    b.check()
    from paper_1209_2137_b200.device import host_checksum

    assert b.checksum() == host_checksum(flat)
