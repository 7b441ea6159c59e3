"""Differential pinning of the oracle against the reference library compiled
from its own sources (oracle/_ref), and of the product's host encoder against
both: identical words, identical decodes, identical accept/reject sets."""
import zlib

import numpy as np
import pytest

import harness as H
import paper_1209_2137_b200 as P
from oracle.pyoracle import RefError
from tests.helpers import F3_NAMES, REF_NAMES, assorted_arrays, chunks_of, random_sorted

# reference what() text -> izg_status (codec_*.cpp throw sites)
WHAT = {
    "chunk: bad original length": 1, "chunk: payload size mismatch": 2,
    "vbyte: truncated stream": 3, "vbyte: value exceeds 32 bits": 4,
    "vbyte: integer longer than 5 bytes": 5, "simdbp128: truncated descriptor": 6,
    "simdbp128: width byte exceeds 32": 7, "simdbp128: truncated payload": 8,
    "fastpfor: truncated page": 9, "fastpfor: bad byte-array offset": 10,
    "fastpfor: truncated byte array": 11, "fastpfor: truncated block metadata": 12,
    "fastpfor: bad block widths": 13, "fastpfor: empty exception list": 14,
    "fastpfor: truncated exception positions": 15,
    "fastpfor: exception position out of range": 16,
    "fastpfor: byte array length mismatch": 17, "fastpfor: missing exception bitset": 18,
    "fastpfor: truncated exception array": 19,
    "fastpfor: packed blocks overrun byte array": 20,
    "fastpfor: exception array exhausted": 21, "fastpfor: packed area size mismatch": 22,
    "bp32: truncated descriptor": 34, "bp32: width byte exceeds 32": 35,
    "bp32: truncated payload": 36, "simple8b: stream exhausted before count": 37,
}


@pytest.mark.parametrize("name", REF_NAMES)
def test_encode_decode_match_reference(oracle, ref, name):
    for arr in assorted_arrays(seed=zlib.crc32(name.encode()) % 997):
        rc = ref.encode_array(name, arr)
        oc = oracle.encode_array(name, arr)
        assert [n for n, _ in rc] == [n for n, _ in oc]
        for (_, a), (_, b) in zip(rc, oc):
            assert np.array_equal(a, b)
        st, out = oracle.decode_array(name, rc)
        assert st == 0 and np.array_equal(out, arr)
        assert np.array_equal(ref.decode_array(name, rc), arr)


@pytest.mark.parametrize("name", REF_NAMES)
def test_host_encoder_bit_exact(native, ref, name):
    codec = P.make_codec(name)
    for arr in assorted_arrays(seed=7 + zlib.crc32(name.encode()) % 991):
        enc = H.encode_array(codec, arr)
        mine = chunks_of(enc)
        theirs = ref.encode_array(name, arr)
        assert [n for n, _ in mine] == [n for n, _ in theirs]
        for (_, a), (_, b) in zip(mine, theirs):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("codec_name", ["simdbp128", "simdfastpfor"])
def test_host_encoder_deltas_every_width(native, ref, codec_name):
    codec = P.make_codec(codec_name)
    rng = np.random.default_rng(5)
    for b in range(33):
        n = 128 * int(rng.integers(1, 12))
        vals = (rng.integers(0, 2**32, size=n, dtype=np.uint64) & ((1 << b) - 1)).astype(np.uint32)
        if b % 3 == 0 and n > 128:  # outliers exercise FastPFOR exceptions
            vals[::37] = rng.integers(0, 2**32, size=len(vals[::37]), dtype=np.uint64)
        e = H.encode_chunks(codec, vals, np.array([0], np.uint64), np.array([n], np.uint32),
                            raw=True)
        mine = e.words[int(e.table["word_off"][0]):][:int(e.table["n_words"][0])]
        assert np.array_equal(mine, ref.encode_deltas(codec_name, vals))


def test_host_encoder_wrapping_matches_reference(native, ref):
    """sums wrap mod 2^32; the reference-side wrapping
    encoder (shim over Codec::encode_deltas) and ours agree."""
    vals, _ = H.gen_arrays("geometric", 4, 65536, 32, seed=3, rate_ppm=100000)
    for name in ("simdfastpfor-s4", "simdbp128-s4"):
        codec = P.make_codec(name)
        for row in vals:
            e = H.encode_array(codec, row, allow_wrap=True)
            mine = chunks_of(e)[0][1]
            assert np.array_equal(mine, ref.encode_chunk_wrapping(name, row))
            assert np.array_equal(ref.decode_array(name, [(len(row), mine)]), row)


def _mutations(payload, rng, reps):
    out = []
    for rep in range(reps):
        p = payload.copy()
        b = p.view(np.uint8)
        for _ in range(1 + rep % 4):
            b[rng.integers(0, len(b))] = rng.integers(0, 256)
        if rep % 5 == 0:
            p = p[:int(rng.integers(0, len(p)))]
        out.append(p)
    return out


@pytest.mark.parametrize("name", REF_NAMES)
def test_corruption_statuses_match_reference(oracle, ref, name):
    """codec_core_test.cpp:221-246 strategy: the oracle's status equals the
    reference's throw (mapped by what()) on every mutated chunk, and accepted
    chunks decode identically."""
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    for n in (700, 2048 + 130, 9000):
        arr = random_sorted(rng, n, 5000)
        payload = ref.encode_array(name, arr)[0][1]
        for p in _mutations(payload, rng, 150):
            st, out = oracle.decode_chunk(name, p, n)
            try:
                expect = ref.decode_array(name, [(n, p)])
                assert st == 0
                assert np.array_equal(out, expect)
            except RefError as e:
                assert e.code == 1, e
                assert st == WHAT[e.what], (e.what, st)


@pytest.mark.parametrize("codec_name", ["simdbp128", "simdfastpfor"])
def test_decode_deltas_corruption_vs_reference(oracle, ref, codec_name):
    rng = np.random.default_rng(99)
    vals = random_sorted(rng, 4096, 3000)
    d = np.diff(vals, prepend=0).astype(np.uint32)
    payload = ref.encode_deltas(codec_name, d)
    for p in _mutations(payload, rng, 200):
        st, out, used = oracle.decode_deltas(codec_name, p, len(d))
        try:
            expect, rused = ref.decode_deltas(codec_name, p, len(d))
            assert st == 0 and used == rused and np.array_equal(out, expect)
        except RefError as e:
            assert st == WHAT[e.what], (e.what, st)


def outlier_sorted(rng, n, rate=0.08):
    gaps = rng.geometric(1 / 6, size=n).astype(np.uint64)
    m = rng.random(n) < rate
    gaps[m] = rng.integers(1 << 10, 1 << 22, size=int(m.sum()))
    return np.minimum(np.cumsum(gaps), 0xFFFFFFFF).astype(np.uint32)


@pytest.mark.parametrize("name", F3_NAMES)
def test_f3_codecs_decode_matches_reference(oracle, ref, name):
    """BP32 / FastPFOR (scalar) / SimplePFOR: the oracle
    decodes reference-encoded arrays exactly, edge lengths and outliers."""
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    arrays = assorted_arrays(seed=zlib.crc32(name.encode()) % 991)
    arrays += [outlier_sorted(rng, n) for n in (128, 4096, 65536, 70000)]
    for arr in arrays:
        st, out = oracle.decode_array(name, ref.encode_array(name, arr))
        assert st == 0 and np.array_equal(out, arr), (name, len(arr))


@pytest.mark.parametrize("name", F3_NAMES)
def test_f3_codecs_corruption_statuses_match_reference(oracle, ref, name):
    rng = np.random.default_rng(zlib.crc32(name.encode()) + 7)
    seen = set()
    for n in (700, 2048 + 130, 9000):
        arr = outlier_sorted(rng, n) if n != 700 else random_sorted(rng, n, 5000)
        payload = ref.encode_array(name, arr)[0][1]
        for p in _mutations(payload, rng, 120):
            st, out = oracle.decode_chunk(name, p, n)
            try:
                expect = ref.decode_array(name, [(n, p)])
                assert st == 0
                assert np.array_equal(out, expect)
            except RefError as e:
                assert e.code == 1, e
                assert st == WHAT[e.what], (e.what, st)
            seen.add(st)
    assert len(seen) >= 3, seen
