"""Pin the oracle (and the product's host encoder) to the reference's own
known-answer tests, and cross-check against the reference
library compiled from source where it is available."""
import numpy as np
import pytest

import harness as H
import paper_1209_2137_b200 as P
from oracle.pyoracle import RefError
from tests import refcases as RC

S = {"ok": 0}


@pytest.mark.parametrize("b", range(33))
def test_vertical_lane_oracle(oracle, b):
    """bitpack_test.cpp:104-119 / acceptance_main.cpp:308-327: pack equals
    the lane-split bit-string oracle; unpack inverts it."""
    rng = np.random.default_rng(3 + b)
    for _ in range(20):
        vals = RC.random_block(rng, 128, b)
        expect = RC.ref_pack_vertical(vals, b)
        got = oracle.pack_vertical128(vals, b)
        assert np.array_equal(got, expect)
        assert np.array_equal(oracle.unpack_vertical128(expect if b else np.zeros(4, np.uint32), b),
                              vals)


def test_vertical_lane_oracle_vs_reference(ref):
    rng = np.random.default_rng(31)
    for b in range(33):
        vals = RC.random_block(rng, 128, b)
        assert np.array_equal(ref.pack_vertical128(vals, b), RC.ref_pack_vertical(vals, b))
        w = RC.ref_pack_vertical(vals, b)
        assert np.array_equal(ref.unpack_vertical128(w if b else np.zeros(4, np.uint32), b), vals)


def test_max_bitwidth(oracle):
    """bitpack_test.cpp:18-28."""
    assert oracle.max_bitwidth([]) == 0
    assert oracle.max_bitwidth([0, 0, 0]) == 0
    assert oracle.max_bitwidth([1]) == 1
    assert oracle.max_bitwidth([3, 4, 1]) == 3
    assert oracle.max_bitwidth([5, 0x80000000]) == 32


def test_delta_examples(oracle):
    """delta_test.cpp:14-26, 43-61, 98-106."""
    d, x = RC.D1_EXAMPLE
    assert list(oracle.delta_decode(1, d)) == x
    assert list(oracle.delta_encode(1, [5, 7, 7, 10])) == [5, 2, 0, 3]
    x4, d4 = RC.D4_EXAMPLE
    assert list(oracle.delta_encode(2, x4)) == d4
    assert list(oracle.delta_decode(2, d4)) == x4
    for n in range(5):
        v = [7 * (i + 1) for i in range(n)]
        assert list(oracle.delta_encode(2, v)) == v
        assert list(oracle.delta_decode(2, v)) == v
    with pytest.raises(ValueError):
        oracle.delta_encode(1, [5, 4])
    with pytest.raises(ValueError):
        oracle.delta_encode(2, [10, 20, 30, 40, 9, 21, 31, 41])
    for mode in (1, 2, 3, 4):
        v = [123456] * 100
        assert list(oracle.delta_decode(mode, oracle.delta_encode(mode, v))) == v


def test_delta_stride4_matches_scalar_loop(oracle, ref):
    """delta_test.cpp:84-96 on the oracle and the reference."""
    rng = np.random.default_rng(12)
    for _ in range(100):
        n = 5 + int(rng.integers(0, 200))
        d = rng.integers(0, 1000, size=n).astype(np.uint32)
        e = d.copy()
        for i in range(4, n):
            e[i] = e[i] + e[i - 4]
        assert np.array_equal(oracle.delta_decode(2, d), e)
        assert np.array_equal(ref.delta(False, True, d), e)


def test_vbyte_goldens(oracle, ref):
    for v, b in RC.VBYTE_GOLDENS:
        assert list(oracle.vbyte_encode([v])) == b
        assert list(ref.vbyte_encode([v])) == b
        st, out, used = oracle.vbyte_decode(b, 1)
        assert st == 0 and int(out[0]) == v and used == len(b)


def test_vbyte_errors(oracle, ref):
    for b, n, code in RC.VBYTE_ERRORS:
        st, _, _ = oracle.vbyte_decode(b, n)
        assert st == code
        with pytest.raises(RefError):
            ref.vbyte_decode(b, n)


def test_fastpfor_width_goldens(oracle, ref):
    """codec_patched_test.cpp:42-72."""
    h = oracle.histogram(RC.WORKED_BLOCK)
    assert h[1] == 3 and h[2] == 10 and h[6] == 3 and h.sum() == 16
    for b, cost in RC.WORKED_COSTS.items():
        assert oracle.cost_bits(h, 16, b) == cost
    assert oracle.choose_width(h, 16) == RC.WORKED_CHOICE
    assert ref.choose_width(h, 16)[:2] == RC.WORKED_CHOICE
    assert oracle.choose_width(oracle.histogram([21] * 128), 128) == (5, 5)
    assert oracle.choose_width(np.zeros(33, np.uint32), 128) == (0, 0)


def test_fastpfor_width_brute_force(oracle, ref):
    """codec_patched_test.cpp:74-109 (brute force, ties toward larger b)."""
    rng = np.random.default_rng(41)
    for _ in range(500):
        h = np.zeros(33, np.uint32)
        maxw = int(rng.integers(0, 33))
        h[:maxw + 1] = rng.integers(0, 40, size=maxw + 1)
        if h.sum() == 0:
            h[0] = 1
        total = int(h.sum())
        maxbits = int(np.nonzero(h)[0].max())
        best_b, best = 0, None
        for b in range(maxbits + 1):
            c = int(h[b + 1:].sum())
            cost = b * total + ((8 + maxbits - b) * c if c else 0)
            if best is None or cost <= best:
                best, best_b = cost, b
        assert oracle.choose_width(h, total) == (best_b, maxbits)
        rb, rm, rc = ref.choose_width(h, total)
        assert (rb, rm, rc) == (best_b, maxbits, best)


def test_simdbp128_goldens(oracle):
    """codec_binpack_test.cpp:102-131."""
    assert list(oracle.encode_deltas("simdbp128", np.zeros(2048, np.uint32))) == [0, 0, 0, 0]
    vals = np.array([7] * 128 + [0x3FF] * 128, np.uint32)
    w = oracle.encode_deltas("simdbp128", vals)
    assert len(w) == 4 + 4 * 3 + 4 * 10
    assert list(w[:4]) == [3 | 10 << 8, 0, 0, 0]
    st, out, used = oracle.decode_deltas("simdbp128", w, 256)
    assert st == 0 and used == len(w) and np.array_equal(out, vals)
    rng = np.random.default_rng(32)
    vals = RC.random_block(rng, 128, 9)
    w = oracle.encode_deltas("simdbp128", vals)
    assert np.array_equal(w[4:], RC.ref_pack_vertical(vals, 9))


def test_simdbp128_corrupt(oracle):
    """codec_binpack_test.cpp:152-164 (and 93-100 on SIMD-BP128)."""
    vals = np.full(128, 255, np.uint32)
    w = oracle.encode_deltas("simdbp128", vals)
    bad = w.copy()
    bad[0] = 40
    assert oracle.decode_deltas("simdbp128", bad, 128)[0] == 7  # width > 32
    assert oracle.decode_deltas("simdbp128", w[:-1], 128)[0] == 8  # truncated payload
    assert oracle.decode_deltas("simdbp128", [], 128)[0] == 6  # truncated descriptor
    assert oracle.decode_deltas("simdbp128", w, 100)[0] == 64  # count % 128


def test_simdfastpfor_worked_page(oracle, ref):
    """codec_patched_test.cpp:274-301: the 32-word golden page."""
    page = RC.worked_page128()
    exp = RC.worked_page_expected_words()
    for w in (oracle.encode_deltas("simdfastpfor", page), ref.encode_deltas("simdfastpfor", page)):
        assert len(w) == exp["size"]
        for k in (0, 9, 12, 13, 14, 15):
            assert int(w[k]) == exp[k], k
        assert np.array_equal(w[1:9], exp["packed_1_9"])
        assert list(w[10:12].view(np.uint8)[:6]) == exp["byte_array"]
        assert np.array_equal(w[16:32], exp["highs_16_32"])
        st, out, used = oracle.decode_deltas("simdfastpfor", w, 128)
        assert st == 0 and used == 32 and np.array_equal(out, page)


def test_simdfastpfor_no_exception_metadata(oracle):
    """codec_patched_test.cpp:303-312 (same byte array for every FastPFOR
    variant): a no-exception block's entry is exactly [b, maxbits]."""
    w = oracle.encode_deltas("simdfastpfor", np.full(128, 5, np.uint32))
    assert int(w[0]) == 13 and int(w[13]) == 2 and int(w[14]) == (3 | 3 << 8)


def test_simdfastpfor_adversarial_pages(oracle, ref):
    """codec_patched_test.cpp:339-358."""
    pages = [np.zeros(128, np.uint32), np.full(128, 0xFFFFFFFF, np.uint32)]
    o = np.ones(256, np.uint32)
    o[200] = 1 << 31
    pages.append(o)
    pages.append(np.array([0xFFFFFFF if i % 2 else 1 for i in range(128)], np.uint32))
    for p in pages:
        w = oracle.encode_deltas("simdfastpfor", p)
        assert np.array_equal(w, ref.encode_deltas("simdfastpfor", p))
        st, out, _ = oracle.decode_deltas("simdfastpfor", w, len(p))
        assert st == 0 and np.array_equal(out, p)


def test_simdfastpfor_decode_errors(oracle):
    """codec_patched_test.cpp:360-384 restated on SIMD-FastPFOR's page (word
    indices shift: the SIMD page is 32 words)."""
    w = oracle.encode_deltas("simdfastpfor", RC.worked_page128())
    assert oracle.decode_deltas("simdfastpfor", [], 128)[0] == 9
    bad = w.copy(); bad[0] = 0
    assert oracle.decode_deltas("simdfastpfor", bad, 128)[0] == 10
    bad[0] = 1000
    assert oracle.decode_deltas("simdfastpfor", bad, 128)[0] == 10
    bad = w.copy(); bad[9] = 1000
    assert oracle.decode_deltas("simdfastpfor", bad, 128)[0] == 11
    bad = w.copy(); bad[11] = 9 | 200 << 8  # position byte 200
    assert oracle.decode_deltas("simdfastpfor", bad, 128)[0] == 16
    bad = w.copy(); bad[13] = 0xFFFFFF  # exception count overruns the payload
    assert oracle.decode_deltas("simdfastpfor", bad, 128)[0] == 19


def test_pipeline_remainder_golden(oracle):
    """codec_core_test.cpp:45-62 on simdbp128: 130 values 3i+1 -> core of 128
    deltas, then the two remainder deltas (3, 3) as VByte 0x83 0x83 in one
    zero-padded word."""
    vals = np.array([3 * i + 1 for i in range(130)], np.uint32)
    payload = oracle.encode_chunk("simdbp128", vals)
    deltas = oracle.delta_encode(1, vals)
    core = oracle.encode_deltas("simdbp128", deltas[:128])
    assert len(payload) == len(core) + 1 and int(payload[-1]) == (0x83 | 0x83 << 8)
    st, out = oracle.decode_chunk("simdbp128", payload, 130)
    assert st == 0 and np.array_equal(out, vals)


def test_pipeline_validation(oracle):
    """codec_core_test.cpp:79-97 (length checks, trailing garbage, empty)."""
    vals = np.array([1, 2, 3], np.uint32)
    for name in ("simdbp128", "simdfastpfor-s4"):
        p = oracle.encode_chunk(name, vals)
        assert oracle.decode_chunk(name, p, 0)[0] == 1
        assert oracle.decode_chunk(name, p, 65537)[0] == 1
        assert oracle.decode_chunk(name, np.append(p, 0), 3)[0] == 2
        assert oracle.decode_chunk(name, [], 3)[0] == 3  # VByte truncated


def test_chunks_independent(oracle, ref):
    """codec_core_test.cpp:64-77 on simdbp128."""
    rng = np.random.default_rng(51)
    vals = np.cumsum(1 + rng.integers(0, 50, size=(1 << 16) + 1000)).astype(np.uint32)
    chunks = ref.encode_array("simdbp128", vals)
    assert len(chunks) == 2
    st, tail = oracle.decode_array("simdbp128", chunks[1:])
    assert st == 0 and np.array_equal(tail, vals[1 << 16:])


@pytest.mark.parametrize("name", ["simdbp128", "simdbp128-s4", "simdfastpfor", "simdfastpfor-s4"])
def test_host_encoder_matches_reference_goldens(native, name):
    """The product's host encoder reproduces the reference goldens above."""
    codec = P.make_codec(name)
    page = RC.worked_page128()
    if name == "simdfastpfor":
        e = H.encode_chunks(codec, page, np.array([0], np.uint64), np.array([128], np.uint32),
                            raw=True)
        w = e.words[int(e.table["word_off"][0]):][:int(e.table["n_words"][0])]
        assert len(w) == 32 and int(w[0]) == 9 and int(w[9]) == 6
    if name == "simdbp128":
        e = H.encode_chunks(codec, np.zeros(2048, np.uint32), np.array([0], np.uint64),
                            np.array([2048], np.uint32), raw=True)
        assert list(e.words[:int(e.table["n_words"][0])]) == [0, 0, 0, 0]
