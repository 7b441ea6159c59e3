"""GPU parity of the two-launch SIMD-FastPFOR path (izg_decode_ws: page index
pass + table-driven decode) against the single fused launch (izg_decode) and
the oracle.

Structural mutations target every metadata field of a page (codec_patched.cpp
:292-416): the byte-array offset A, the byte-array length L, entry widths and
counts, exception positions, the exception bitset and the per-width counts,
and truncations at each region boundary.  Bar: identical per-chunk statuses
and words consumed on both paths and in the oracle; identical outputs for
every chunk that decodes.
"""
import zlib

import numpy as np
import pytest

import harness as H
import paper_1209_2137_b200 as P
from tests.helpers import random_sorted

pytestmark = pytest.mark.gpu

FP_NAMES = ["simdfastpfor", "simdfastpfor-s4", "simdfastpfor-d2", "simdfastpfor-dm"]


def outlier_array(rng, n, rate=0.08):
    gaps = rng.geometric(1 / 6, size=n).astype(np.uint64)
    m = rng.random(n) < rate
    gaps[m] = rng.integers(1 << 10, 1 << 22, size=int(m.sum()))
    return np.minimum(np.cumsum(gaps), 0xFFFFFFFF).astype(np.uint32)


def page_fields(p):
    """(A, L, entry starts, exception-entry starts, directory word) of a page."""
    A = int(p[0])
    L = int(p[A])
    ba = p[A + 1:].view(np.uint8)
    starts, exc = [], []
    s = 0
    while s + 2 <= L:
        b, mb = int(ba[s]), int(ba[s + 1])
        starts.append(s)
        if mb > b:
            exc.append(s)
            s += 3 + int(ba[s + 2])
        else:
            s += 2
    return A, L, starts, exc, A + 1 + (L + 3) // 4


def mutations(rng, p):
    """Structural variants of one page payload (uint32 array)."""
    A, L, starts, exc, bit_w = page_fields(p)
    out = []

    def var(f):
        q = p.copy()
        f(q, q[A + 1:].view(np.uint8))
        out.append(q)

    for d in (-1, 1, 5):
        var(lambda q, ba, d=d: q.__setitem__(0, (A + d) & 0xFFFFFFFF))
        var(lambda q, ba, d=d: q.__setitem__(A, (L + d) & 0xFFFFFFFF))
    for s in (rng.choice(starts, size=min(6, len(starts)), replace=False) if starts else []):
        var(lambda q, ba, s=s: ba.__setitem__(s, (int(ba[s]) + 1) % 40))      # b
        var(lambda q, ba, s=s: ba.__setitem__(s + 1, (int(ba[s + 1]) + 3) % 40))  # maxbits
    for s in (rng.choice(exc, size=min(6, len(exc)), replace=False) if exc else []):
        c = int(p[A + 1:].view(np.uint8)[s + 2])
        var(lambda q, ba, s=s: ba.__setitem__(s + 2, c + 1))                   # count
        var(lambda q, ba, s=s: ba.__setitem__(s + 2, max(c - 1, 0)))
        var(lambda q, ba, s=s: ba.__setitem__(s + 3 + int(rng.integers(0, c)),
                                              128 + int(rng.integers(0, 128))))  # position
    if bit_w < len(p):
        bits = int(p[bit_w])
        for k in (0, 3, 9):
            var(lambda q, ba, k=k: q.__setitem__(bit_w, bits ^ (1 << k)))
        if bit_w + 1 < len(p):
            for d in (-1, 1, 200):
                var(lambda q, ba, d=d: q.__setitem__(bit_w + 1, (int(p[bit_w + 1]) + d) & 0xFFFFFFFF))
    for cut in {0, 1, A, A + 1, bit_w, bit_w + 1, bit_w + 2, len(p) - 1}:
        if 0 <= cut < len(p):
            out.append(p[:cut].copy())
    return out


def corpus(name, seed):
    rng = np.random.default_rng(seed)
    codec = P.make_codec(name)
    payloads, counts = [], []
    for n in (128, 700, 2048 + 130, 9000, 65536):
        arr = outlier_array(rng, n)
        p = H.encode_array(codec, arr)
        payload = p.words[int(p.table["word_off"][0]):][:int(p.table["n_words"][0])].copy()
        payloads.append(payload)
        counts.append(n)
        for q in mutations(rng, payload):
            payloads.append(q)
            counts.append(n)
    return codec, payloads, counts


def both_paths(codec, enc, raw=False):
    """(fused one-warp, workspace path) results; the workspace path of a small
    batch is the split kernel, and the one-warp indexed kernel (workspace of
    the page index only) must agree with both."""
    res = []
    for indexed, split in ((False, True), (True, False), (True, True)):
        b = P.DeviceBatch(codec, enc, raw=raw, indexed=indexed, split=split)
        assert (b.workspace is not None) == indexed
        b.decode()
        res.append((b.statuses(), b.output(), b.consumed[:b.n_chunks].cpu().numpy()))
    (s0, o0, u0), (s1, o1, u1), (s2, o2, u2) = res
    assert np.array_equal(s0, s1) and np.array_equal(s1, s2)
    assert np.array_equal(u1, u2)
    for i in np.nonzero(s1 == 0)[0]:
        a = int(enc.table["out_off"][i])
        n = int(enc.table["n"][i])
        assert np.array_equal(o1[a:a + n], o2[a:a + n]), i
    return res[0], res[2]


@pytest.mark.parametrize("name", FP_NAMES)
def test_structural_mutations_array(cuda, oracle, name):
    codec, payloads, counts = corpus(name, zlib.crc32(name.encode()))
    enc = P.layout(codec, payloads, counts)
    (s0, o0, _), (s1, o1, _) = both_paths(codec, enc)
    assert np.array_equal(s0, s1), np.nonzero(s0 != s1)[0][:10]
    n_err = 0
    for i, (p, n) in enumerate(zip(payloads, counts)):
        ost, oout = oracle.decode_chunk(name, p, n)
        assert s1[i] == ost, (i, s1[i], ost)
        n_err += ost != 0
        if ost == 0:
            o = int(enc.table["out_off"][i])
            assert np.array_equal(o1[o:o + n], oout), i
            assert np.array_equal(o0[o:o + n], oout), i
    assert n_err > len(payloads) // 2  # the corpus really is mostly corrupt
    # the corpus reaches many FastPFOR status classes
    seen = set(int(x) for x in s1) & set(range(9, 23))
    assert len(seen) >= 6, seen


@pytest.mark.parametrize("name", ["simdfastpfor", "simdfastpfor-s4"])
def test_structural_mutations_raw(cuda, oracle, name):
    """decode_deltas (codec.h:36-40): statuses and words consumed."""
    rng = np.random.default_rng(7)
    codec = P.make_codec(name)
    payloads, counts = [], []
    for n in (128, 1024, 65536):
        deltas = outlier_array(rng, n) % (1 << 20)
        p = oracle.encode_deltas(name, deltas)
        payloads.append(p)
        counts.append(n)
        for q in mutations(rng, p):
            payloads.append(q)
            counts.append(n)
    enc = P.layout(codec, payloads, counts)
    (s0, o0, u0), (s1, o1, u1) = both_paths(codec, enc, raw=True)
    assert np.array_equal(s0, s1)
    assert np.array_equal(u0, u1)
    for i, (p, n) in enumerate(zip(payloads, counts)):
        ost, oout, used = oracle.decode_deltas(name, p, n)
        assert s1[i] == ost, (i, s1[i], ost)
        if ost == 0:
            assert u1[i] == used
            o = int(enc.table["out_off"][i])
            assert np.array_equal(o1[o:o + n], oout), i


@pytest.mark.parametrize("name", FP_NAMES)
def test_random_byte_fuzz_both_paths(cuda, name):
    codec = P.make_codec(name)
    rng = np.random.default_rng(zlib.crc32(name.encode()) + 1)
    payloads, counts = [], []
    for rep in range(400):
        n = int(rng.choice([300, 4096, 20000]))
        arr = outlier_array(rng, n) if rep % 2 else random_sorted(rng, n, 3000)
        e = H.encode_array(codec, arr)
        p = e.words[int(e.table["word_off"][0]):][:int(e.table["n_words"][0])].copy()
        b = p.view(np.uint8)
        for _ in range(1 + rep % 3):
            b[rng.integers(0, len(b))] = rng.integers(0, 256)
        payloads.append(p)
        counts.append(n)
    enc = P.layout(codec, payloads, counts)
    (s0, o0, _), (s1, o1, _) = both_paths(codec, enc)
    assert np.array_equal(s0, s1)
    for i, n in enumerate(counts):
        if s1[i] == 0:
            o = int(enc.table["out_off"][i])
            assert np.array_equal(o0[o:o + n], o1[o:o + n]), i


def test_workspace_too_small_falls_back_to_fused(cuda):
    """izg_decode_ws with an undersized workspace is exactly izg_decode."""
    import torch

    from paper_1209_2137_b200 import _native as N

    codec = P.make_codec("simdfastpfor-s4")
    rng = np.random.default_rng(3)
    arr = outlier_array(rng, 3 * 65536)
    enc = H.encode_array(codec, arr)
    b = P.DeviceBatch(codec, enc, indexed=False)
    ws = torch.empty(64, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    rc = N.lib().izg_decode_ws(codec.codec, codec.delta, N.ptr(b.words), N.ptr(b.table),
                               b.n_chunks, N.ptr(b.out), N.ptr(b.status), None, N.ptr(ws), 64,
                               s.cuda_stream)
    assert rc == N.SUCCESS
    b.check()
    assert np.array_equal(b.output(), arr)
    # large batches: the page index only (SIMD-FastPFOR), nothing for SIMD-BP128;
    # small ones add the split kernel's look-back state (test_gpu_split.py)
    n = 1 << 14
    assert N.lib().izg_decode_workspace_size(0, n) == 0
    assert N.lib().izg_decode_workspace_size(1, n) == n * (16 + 128 + 512 * 16 + 1024)
    assert N.lib().izg_decode_workspace_size(1, 100) > 100 * (16 + 128 + 512 * 16 + 1024)


_BIG = r'''
import sys
sys.path.insert(0, {root!r})
import torch
from oracle.pyoracle import Oracle
from tests import test_gpu_indexed as T
O = Oracle()
for name in T.FP_NAMES:
    T.test_structural_mutations_array(torch, O, name)
    T.test_random_byte_fuzz_both_paths(torch, name)
for name in ["simdfastpfor", "simdfastpfor-s4"]:
    T.test_structural_mutations_raw(torch, O, name)
print("ok")
'''


def test_large_batch_shape():
    """The indexed decode's large-batch shape (24 warps at 80 registers, taken
    from IZG_BIG_IDX_BATCH pages on) forced onto the small batches of this
    file: statuses and outputs against the oracle and the fused path."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, IZG_BIG_IDX_BATCH="1", IZG_SPLIT="0", IZG_TEAM="0")
    r = subprocess.run([sys.executable, "-c", _BIG.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


@pytest.mark.parametrize("env", [{"IZG_INDEX_LANES_MIN": "0", "IZG_SPLIT": "0", "IZG_TEAM": "0"},
                                 {"IZG_INDEX_LANES_MIN": "0", "IZG_SPLIT": "1"}],
                         ids=["indexed", "split"])
def test_lane_index_pass(env):
    """The lane-per-page index pass (fp_index_lanes_kernel, taken from
    IZG_INDEX_LANES_MIN pages on) forced onto the small batches of this file
    — every structural mutation, random fuzz and raw case — in front of the
    indexed decode and of the split decode: statuses and outputs against the
    oracle and the fused path, as with the warp-per-page pass."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _BIG.format(root=root)],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


_LARGE = r'''
import sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P
from paper_1209_2137_b200.device import host_checksum
codec = P.make_codec("simdfastpfor-s4")
for model, count, d, rate in [("cluster", 8192, (20, 29), 0), ("geometric", 2048, 32, 100000)]:
    vals, _ = H.gen_arrays(model, count, 65536, d, seed=11, rate_ppm=rate)
    flat = vals.reshape(-1)
    enc = H.encode_chunks(codec, flat, np.arange(count, dtype=np.uint64) * 65536,
                          np.full(count, 65536, np.uint32), allow_wrap=model == "geometric")
    want = host_checksum(flat)
    b = P.DeviceBatch(codec, enc)
    for _ in range(4):   # the failure this guards against depended on memory load
        b.out.zero_()
        b.decode()
        torch.cuda.synchronize()
        b.check()
        assert b.checksum() == want
print("ok")
'''


@pytest.mark.parametrize("team", ["0", "1"], ids=["warp-per-page", "team"])
def test_lane_index_pass_large_batch(cuda, team):
    """The lane-per-page index pass on batches large enough to load the memory
    system (8,192 C5 pages, 2,048 C4 pages at 10 % outliers): its cp.async
    rings once let a late copy land on a refilled slot, which only showed
    under load.  Device checksum against the generated arrays, repeatedly."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, IZG_INDEX_LANES_MIN="0", IZG_SPLIT="0", IZG_TEAM=team)
    r = subprocess.run([sys.executable, "-c", _LARGE.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-1000:] + r.stderr[-3000:]


@pytest.mark.parametrize("name", ["simdfastpfor-s4", "simdfastpfor", "simdbp128-s4"])
def test_decode_phases_equal_one_call(cuda, name):
    """izg_decode_ws_phase: the page index pass (phase 1) on a side stream,
    then the decode (phase 2), gives izg_decode_ws's outputs, statuses and
    words consumed — including under corruption; codecs without an index
    pass do nothing in phase 1 and everything in phase 2."""
    torch = cuda
    codec = P.make_codec(name)
    rng = np.random.default_rng(77)
    for count in (40, 3000):  # split-decode and indexed-decode batch sizes
        vals = [random_sorted(rng, 65536, int(rng.integers(1, 3000))) for _ in range(count)]
        flat = np.concatenate(vals)
        enc = H.encode_chunks(codec, flat, np.arange(count, dtype=np.uint64) * 65536,
                              np.full(count, 65536, np.uint32))
        w = enc.words.copy()
        for _ in range(5):  # a few corrupted pages
            t = enc.table[int(rng.integers(0, count))]
            w[int(t["word_off"]) + int(rng.integers(0, int(t["n_words"])))] ^= np.uint32(1 << 7)
        bad = P.Encoded(w, enc.table)
        one = P.DeviceBatch(codec, bad)
        two = P.DeviceBatch(codec, bad)
        one.decode()
        side = torch.cuda.Stream()
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        side.wait_event(ev)
        two.decode_phase(1, side)
        ev2 = torch.cuda.Event()
        ev2.record(side)
        torch.cuda.current_stream().wait_event(ev2)
        two.decode_phase(2)
        torch.cuda.synchronize()
        assert np.array_equal(one.statuses(), two.statuses())
        ok = one.statuses() == 0
        assert ok.sum() >= count - 5
        o1, o2 = one.output().reshape(count, 65536), two.output().reshape(count, 65536)
        assert np.array_equal(o1[ok], o2[ok])
        assert np.array_equal(one.consumed[:count].cpu().numpy(), two.consumed[:count].cpu().numpy())
