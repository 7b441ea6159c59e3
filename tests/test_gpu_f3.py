"""GPU parity for the scalar-group codecs of SURVEY.md §8 f3 — BP32
(codec_binpack.cpp:17-60), FastPFOR with scalar exception arrays and
SimplePFOR with a Simple-8b stream of exception highs (codec_patched.cpp
:292-417, PatchStorage::scalar_arrays / simple8b) — against the reference
(compiled from source) and the oracle.  Inputs are encoded by the
reference itself; the bar is bit-exact outputs and identical per-chunk
statuses, through the host entry point and the device entry point (both
run the fused page kernel for these codecs).
"""
import zlib

import numpy as np
import pytest

import paper_1209_2137_b200 as P
from tests.helpers import assorted_arrays, random_sorted

pytestmark = pytest.mark.gpu

NAMES = ["bp32", "bp32-s4", "fastpfor", "fastpfor-s4", "simplepfor", "simplepfor-s4"]


def outlier_sorted(rng, n, rate=0.08):
    gaps = rng.geometric(1 / 6, size=n).astype(np.uint64)
    m = rng.random(n) < rate
    gaps[m] = rng.integers(1 << 10, 1 << 22, size=int(m.sum()))
    return np.minimum(np.cumsum(gaps), 0xFFFFFFFF).astype(np.uint32)


def ref_encoded(ref, codec, arrays):
    payloads, counts = [], []
    for a in arrays:
        for n, p in ref.encode_array(codec.name, a):
            payloads.append(p)
            counts.append(n)
    return P.layout(codec, payloads, counts), payloads, counts


def decode_both(codec, enc, raw=False):
    """(host path = izg_decode_host, fused device path) outputs + statuses."""
    got, st = P.decode_array(codec, enc, raw=raw, return_status=True)
    b = P.DeviceBatch(codec, enc, raw=raw, indexed=False)
    b.decode()
    return (got, st), (b.output(), b.statuses(), b.consumed[:b.n_chunks].cpu().numpy())


@pytest.mark.parametrize("name", NAMES)
def test_reference_encoded_arrays(cuda, ref, name):
    codec = P.make_codec(name)
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    arrays = assorted_arrays(seed=zlib.crc32(name.encode()) % 313)
    arrays += [outlier_sorted(rng, n) for n in (128, 4096, 65536, 3 * 65536 + 77)]
    enc, _, _ = ref_encoded(ref, codec, arrays)
    (h, hs), (d, ds, _) = decode_both(codec, enc)
    flat = np.concatenate(arrays)
    assert not hs.any() and not ds.any()
    assert np.array_equal(h, flat)
    assert np.array_equal(d, flat)


@pytest.mark.parametrize("name", ["bp32", "fastpfor", "simplepfor"])
def test_decode_deltas_every_width(cuda, ref, name):
    """decode_deltas (raw) at every width 0..32, words consumed included."""
    codec = P.make_codec(name)
    rng = np.random.default_rng(5)
    payloads, counts, deltas = [], [], []
    for b in range(33):
        n = 128 * int(rng.integers(1, 20))
        v = (rng.integers(0, 2**32, size=n, dtype=np.uint64) & ((1 << b) - 1)).astype(np.uint32)
        if b and name != "bp32":  # a few wide values: exceptions at every width
            v[rng.integers(0, n, size=3)] |= np.uint32(1 << (b - 1))
        payloads.append(ref.encode_deltas(name, v))
        counts.append(n)
        deltas.append(v)
    enc = P.layout(codec, payloads, counts)
    (h, hs), (d, ds, used) = decode_both(codec, enc, raw=True)
    assert not hs.any() and not ds.any()
    flat = np.concatenate(deltas)
    assert np.array_equal(h, flat) and np.array_equal(d, flat)
    assert list(used) == [len(p) for p in payloads]


@pytest.mark.parametrize("name", NAMES)
def test_mutation_fuzz_matches_oracle(cuda, ref, oracle, name):
    codec = P.make_codec(name)
    rng = np.random.default_rng(zlib.crc32(name.encode()) + 3)
    payloads, counts = [], []
    for rep in range(300):
        n = int(rng.choice([700, 2048 + 130, 9000]))
        arr = outlier_sorted(rng, n) if rep % 2 else random_sorted(rng, n, 5000)
        p = ref.encode_array(name, arr)[0][1].copy()
        b = p.view(np.uint8)
        for _ in range(1 + rep % 4):
            b[rng.integers(0, len(b))] = rng.integers(0, 256)
        if rep % 5 == 0:
            p = p[:int(rng.integers(0, len(p)))]
        payloads.append(p)
        counts.append(n)
    enc = P.layout(codec, payloads, counts)
    (h, hs), (d, ds, _) = decode_both(codec, enc)
    assert np.array_equal(hs, ds)
    for i, (p, n) in enumerate(zip(payloads, counts)):
        ost, oout = oracle.decode_chunk(name, p, n)
        assert hs[i] == ost, (i, hs[i], ost)
        if ost == 0:
            o = int(enc.table["out_off"][i])
            assert np.array_equal(h[o:o + n], oout), i
            assert np.array_equal(d[o:o + n], oout), i


@pytest.mark.parametrize("name", ["fastpfor-s4", "simplepfor-s4"])
def test_page_structural_mutations(cuda, oracle, name):
    """Every page field of a scalar-group page (the SIMD-FastPFOR structural
    corpus of test_gpu_indexed, reused: for SimplePFOR the "bitset" and
    "count" words are the first Simple-8b word), both decode paths."""
    from tests.test_gpu_indexed import mutations

    codec = P.make_codec(name)
    rng = np.random.default_rng(17)
    payloads, counts = [], []
    for n in (128, 700, 9000, 65536):
        from oracle.pyoracle import Reference

        p = Reference().encode_array(name, outlier_sorted(rng, n))[0][1]
        payloads.append(p)
        counts.append(n)
        for q in mutations(rng, p):
            payloads.append(q)
            counts.append(n)
    enc = P.layout(codec, payloads, counts)
    (h, hs), (d, ds, _) = decode_both(codec, enc)
    assert np.array_equal(hs, ds)
    for i, (p, n) in enumerate(zip(payloads, counts)):
        ost, oout = oracle.decode_chunk(name, p, n)
        assert hs[i] == ost, (i, hs[i], ost)
        if ost == 0:
            o = int(enc.table["out_off"][i])
            assert np.array_equal(h[o:o + n], oout)
