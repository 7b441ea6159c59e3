"""GPU parity: the fused sm_100a decoder vs the oracle and the reference.

Bar: bit-exact outputs and identical per-chunk statuses (integer work).
All calls go through the C ABI (izg_decode_host / izg_decode).
"""
import zlib

import numpy as np
import pytest

import harness as H
import paper_1209_2137_b200 as P
from tests.helpers import (ALL_NAMES, REF_NAMES, assorted_arrays, chunks_of, misplace,
                           random_sorted)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ALL_NAMES)
def test_roundtrip_assorted(cuda, oracle, name):
    codec = P.make_codec(name)
    for arr in assorted_arrays(seed=zlib.crc32(name.encode()) % 1000):
        enc = H.encode_array(codec, arr)
        st, expect = oracle.decode_array(name, chunks_of(enc))
        assert st == 0 and np.array_equal(expect, arr)
        got = P.decode_array(codec, enc)
        assert np.array_equal(got, arr), (name, len(arr))


@pytest.mark.parametrize("name", REF_NAMES)
def test_reference_encoded_buffers_decode(cuda, ref, name):
    """Buffers produced by the CPU reference decode on the GPU."""
    codec = P.make_codec(name)
    rng = np.random.default_rng(5)
    for n in [1, 129, 2049, 65536, 65537, 131072 + 77]:
        arr = random_sorted(rng, n, 5000)
        chunks = ref.encode_array(name, arr)
        enc = P.layout(codec, [p for _, p in chunks], [c for c, _ in chunks])
        got = P.decode_array(codec, enc)
        assert np.array_equal(got, ref.decode_array(name, chunks))
        assert np.array_equal(got, arr)


@pytest.mark.parametrize("name", ALL_NAMES)
@pytest.mark.parametrize("word_phase,out_phase", [(1, 0), (2, 3), (3, 1), (0, 2)])
def test_unaligned_placement(cuda, name, word_phase, out_phase):
    codec = P.make_codec(name)
    rng = np.random.default_rng(word_phase * 7 + out_phase)
    arrs = [random_sorted(rng, n, 3000) for n in (70000, 300, 4096 + 5)]
    for arr in arrs:
        enc = misplace(H.encode_array(codec, arr), word_phase, out_phase)
        got = P.decode_array(codec, enc)
        assert np.array_equal(got[out_phase:], arr)


@pytest.mark.parametrize("codec_name", ["simdbp128", "simdfastpfor"])
def test_decode_deltas_every_width(cuda, ref, codec_name):
    """Codec::decode_deltas at every width b = 0..32 (C2 shape, smaller)."""
    codec = P.make_codec(codec_name)
    rng = np.random.default_rng(11)
    payloads, counts, expect = [], [], []
    for b in range(33):
        n = 128 * int(rng.integers(1, 40))
        vals = (rng.integers(0, 2**32, size=n, dtype=np.uint64) &
                ((1 << b) - 1)).astype(np.uint32)
        w = ref.encode_deltas(codec_name, vals)
        payloads.append(w)
        counts.append(n)
        expect.append(vals)
    enc = P.layout(codec, payloads, counts)
    got = P.decode_array(codec, enc, raw=True)
    assert np.array_equal(got, np.concatenate(expect))


def test_device_batch_consumed_words(cuda, ref):
    """decode_deltas returns words consumed (codec.h:36-40)."""
    codec = P.make_codec("simdbp128")
    rng = np.random.default_rng(12)
    payloads, counts = [], []
    for k in range(20):
        vals = (rng.integers(0, 1 << (k + 3), size=128 * (k + 1))).astype(np.uint32)
        payloads.append(ref.encode_deltas("simdbp128", vals))
        counts.append(len(vals))
    enc = P.layout(codec, [np.concatenate([p, np.zeros(3, np.uint32)]) for p in payloads],
                   counts)
    b = P.DeviceBatch(codec, enc, raw=True)
    b.decode()
    b.check()
    assert list(b.consumed[:len(counts)].cpu().numpy()) == [len(p) for p in payloads]


def test_chunk_length_and_count_errors(cuda):
    codec = P.make_codec("simdbp128-s4")
    enc = H.encode_array(codec, np.arange(1000, dtype=np.uint32))
    bad = P.Encoded(enc.words.copy(), enc.table.copy())
    bad.table["n"][0] = 0
    _, st = P.decode_array(codec, bad, return_status=True)
    assert st[0] == 1  # codec.cpp:43-44
    bad.table["n"][0] = 65537
    bad.table["out_off"][0] = 0
    out, st = P.decode_array(codec, P.Encoded(bad.words, bad.table), return_status=True)
    assert st[0] == 1
    raw = P.Encoded(enc.words.copy(), enc.table.copy())
    raw.table["n"][0] = 100
    _, st = P.decode_array(codec, raw, raw=True, return_status=True)
    assert st[0] == 64  # count % 128 (codec_binpack.cpp:13-14)


@pytest.mark.parametrize("name", ALL_NAMES)
def test_mutation_fuzz_matches_oracle(cuda, oracle, name):
    """codec_core_test.cpp:221-246 strategy on the GPU: random byte
    mutations and truncations; every chunk's status and (when OK) output
    must equal the oracle's."""
    codec = P.make_codec(name)
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    base_arrays = [random_sorted(rng, n, 5000) for n in (700, 2048 + 130, 9000)]
    payloads, counts = [], []
    for rep in range(300):
        arr = base_arrays[rep % 3]
        p = chunks_of(H.encode_array(codec, arr))[0][1].copy()
        b = p.view(np.uint8)
        for _ in range(1 + rep % 4):
            b[rng.integers(0, len(b))] = rng.integers(0, 256)
        if rep % 5 == 0:
            p = p[:int(rng.integers(0, len(p)))]
        payloads.append(p)
        counts.append(len(arr))
    enc = P.layout(codec, payloads, counts)
    got, st = P.decode_array(codec, enc, return_status=True)
    for i, (p, n) in enumerate(zip(payloads, counts)):
        ost, oout = oracle.decode_chunk(name, p, n)
        assert st[i] == ost, (i, st[i], ost)
        if ost == 0:
            o = int(enc.table["out_off"][i])
            assert np.array_equal(got[o:o + n], oout), i


@pytest.mark.parametrize("name", REF_NAMES)
def test_mutation_fuzz_accept_reject_matches_reference(cuda, ref, name):
    codec = P.make_codec(name)
    rng = np.random.default_rng(54)
    arr = random_sorted(rng, 700, 5000)
    payload = ref.encode_array(name, arr)[0][1]
    payloads = []
    for rep in range(200):
        p = payload.copy()
        b = p.view(np.uint8)
        for _ in range(1 + rep % 4):
            b[rng.integers(0, len(b))] = rng.integers(0, 256)
        payloads.append(p)
    enc = P.layout(codec, payloads, [700] * len(payloads))
    got, st = P.decode_array(codec, enc, return_status=True)
    from oracle.pyoracle import RefError

    for i, p in enumerate(payloads):
        try:
            expect = ref.decode_array(name, [(700, p)])
        except RefError:
            expect = None
        if expect is None:
            assert st[i] != 0, i
        else:
            assert st[i] == 0, i
            assert np.array_equal(got[700 * i:700 * (i + 1)], expect)


@pytest.mark.parametrize("name", ["simdbp128-s4", "simdfastpfor-s4"])
def test_device_checksum_large_batch(cuda, name):
    """Size-independent property at a C1-like size: device checksum of the
    decoded batch equals the checksum of the generated input."""
    from paper_1209_2137_b200.device import host_checksum

    codec = P.make_codec(name)
    vals, _ = H.gen_arrays("cluster", 256, 65536, 29, seed=1234)
    flat = vals.reshape(-1)
    offs = np.arange(256, dtype=np.uint64) * 65536
    enc = H.encode_chunks(codec, flat, offs, np.full(256, 65536, np.uint32))
    b = P.DeviceBatch(codec, enc)
    b.decode()
    b.check()
    assert b.checksum() == host_checksum(flat)


_GROUP = r'''
import sys
sys.path.insert(0, {root!r})
import torch
from oracle.pyoracle import Oracle
from tests import test_gpu_parity as T
O = Oracle()
for name in ["simdbp128", "simdbp128-s4", "simdbp128-d2", "simdbp128-dm"]:
    T.test_roundtrip_assorted(torch, O, name)
    T.test_mutation_fuzz_matches_oracle(torch, O, name)
    T.test_unaligned_placement(torch, name, 2, 3)
print("ok")
'''


@pytest.mark.parametrize("kw", [1, 2, 4, 8])
def test_bp128_warps_per_chunk(kw):
    """SIMD-BP128 without the split kernel runs KW warps per chunk on small
    batches (csrc/group.cuh, iterations round robin, mailbox carry): every
    KW, forced with IZG_GROUP (1 = the one-warp kernel), against the oracle
    — outputs and statuses under mutation fuzz, unaligned placements."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, IZG_GROUP=str(kw), IZG_SPLIT="0", IZG_CTA="0")
    r = subprocess.run([sys.executable, "-c", _GROUP.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


def test_host_decode_many_tiny_chunks(cuda, ref):
    """izg_decode_host with more than 2^20 chunks (1-integer arrays, as short
    posting lists give): the reference's decode_array accepts any number of
    chunks, so must the host path (it cuts pieces by chunk count too)."""
    codec = P.make_codec("simdbp128-s4")
    n = (1 << 20) + 4097
    vals = np.random.default_rng(8).integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    enc = H.encode_chunks(codec, vals, np.arange(n, dtype=np.uint64), np.ones(n, np.uint32))
    got = P.decode_array(codec, enc)
    assert np.array_equal(got, vals)
    # spot-check the payload words against the reference encoder
    for i in (0, n // 2, n - 1):
        chunks = ref.encode_array("simdbp128-s4", vals[i:i + 1])
        t = enc.table[i]
        assert np.array_equal(chunks[0][1], enc.words[int(t["word_off"]):][:int(t["n_words"])])


def test_host_decode_leaves_gaps_untouched(cuda):
    """Outputs placed with gaps between chunks: izg_decode_host copies back
    only the decoded ranges, the caller's other words stay as they were."""
    import ctypes as C  # noqa: F401

    codec = P.make_codec("simdfastpfor-s4")
    rng = np.random.default_rng(12)
    arrs = [random_sorted(rng, n, 1000) for n in (70000, 300, 4096 + 5, 65536)]
    encs = [H.encode_array(codec, a) for a in arrs]
    payloads, counts, outs = [], [], []
    pos = 7
    for e in encs:
        for t in e.table:
            payloads.append(e.words[int(t["word_off"]):int(t["word_off"]) + int(t["n_words"])])
            counts.append(int(t["n"]))
            outs.append(pos)
            pos += int(t["n"]) + 1000  # a gap after every chunk
    enc = P.layout(codec, payloads, counts, np.array(outs, dtype=np.uint64))
    L = P._native.lib()
    out = np.full(pos, 0xA5A5A5A5, dtype=np.uint32)
    st = np.zeros(len(counts), np.int32)
    rc = L.izg_decode_host(codec.codec, codec.delta, P._native.ptr(enc.words), len(enc.words),
                           P._native.ptr(enc.table), len(enc.table), P._native.ptr(out), len(out),
                           P._native.ptr(st))
    assert rc == 0 and not st.any()
    mask = np.zeros(pos, bool)
    for o, n in zip(outs, counts):
        mask[o:o + n] = True
    assert np.all(out[~mask] == 0xA5A5A5A5)
    assert np.array_equal(out[mask], np.concatenate(arrs))
