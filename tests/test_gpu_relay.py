"""The SIMD-BP128 relay kernel (csrc/relay.cuh: chunks cut into segments of
whole meta-blocks, (segment, chunk) tasks claimed level by level, each task
reading the payload position, the prefix-sum carry and the first error its
predecessor published, then decoding once through the one-warp core).

Batches of 2,432 .. 14,208 chunks take it by default when a workspace is
given; IZG_RELAY=1 (read once per process, hence subprocesses) forces it
onto the parity suites, where batches are small and every task beyond the
first of a chunk really waits for its predecessor.  Outputs and statuses
against the oracle and the reference: every array mode and the raw mode,
edge lengths, VByte remainders, unaligned placements, mutation fuzz (first
error in stream order), reference-encoded BASELINE config shapes, every
segment count, and a default-routed ragged batch of 4,096 chunks against
the one-warp kernel."""
import os
import subprocess
import sys

import numpy as np
import pytest

import harness as H
import paper_1209_2137_b200 as P
from paper_1209_2137_b200.codec import Encoded
from tests.helpers import random_sorted

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r'''
import sys
sys.path.insert(0, {root!r})
import torch
from oracle.pyoracle import Oracle, Reference
from tests import test_gpu_parity as T
from tests import test_gpu_relay as RL
O, R = Oracle(), Reference()
for name in ["simdbp128", "simdbp128-s4", "simdbp128-d2", "simdbp128-dm"]:
    T.test_roundtrip_assorted(torch, O, name)
    for wp, op in [(1, 0), (2, 3), (0, 2)]:
        T.test_unaligned_placement(torch, name, wp, op)
    T.test_mutation_fuzz_matches_oracle(torch, O, name)
    RL.corruption_vs_one_warp(name)
for name in ["simdbp128", "simdbp128-s4"]:
    T.test_reference_encoded_buffers_decode(torch, R, name)
    T.test_mutation_fuzz_accept_reject_matches_reference(torch, R, name)
RL.raw_chunks_longer_than_the_levels()
T.test_decode_deltas_every_width(torch, R, "simdbp128")
T.test_device_batch_consumed_words(torch, R)
T.test_chunk_length_and_count_errors(torch)
T.test_device_checksum_large_batch(torch, "simdbp128-s4")
print("ok")
'''


def _run(env, code, timeout=900):
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), \
        r.stdout[-2000:] + r.stderr[-4000:]


def corruption_vs_one_warp(name, trials=25):
    """Bit flips in multi-segment chunks: the relay reports exactly the
    one-warp kernel's status per chunk and identical output where it decodes
    (called inside the forced subprocess; DeviceBatch(indexed=False) runs
    izg_decode, which has no workspace and so never takes the relay)."""
    codec = P.make_codec(name)
    rng = np.random.default_rng(23)
    arrays = [random_sorted(rng, 65536, 40) for _ in range(3)] + \
             [random_sorted(rng, n, 9) for n in (30001, 2048, 2047, 127, 1)]
    flat = np.concatenate(arrays).astype(np.uint32)
    counts = np.array([len(a) for a in arrays], np.uint32)
    offs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64)
    enc = H.encode_chunks(codec, flat, offs, counts)
    for trial in range(trials):
        w = enc.words.copy()
        for _ in range(int(rng.integers(0, 4))):
            c = int(rng.integers(0, len(enc.table)))
            off, nw = int(enc.table["word_off"][c]), int(enc.table["n_words"][c])
            w[off + int(rng.integers(0, nw))] ^= np.uint32(1) << np.uint32(rng.integers(0, 32))
        bad = Encoded(w, enc.table)
        a = P.DeviceBatch(codec, bad)
        b = P.DeviceBatch(codec, bad, indexed=False)
        assert a.workspace is not None
        a.decode()
        b.decode()
        sa, sb = a.statuses(), b.statuses()
        assert np.array_equal(sa, sb), (name, trial, sa, sb)
        ca = a.consumed[:a.n_chunks].cpu().numpy()
        cb = b.consumed[:b.n_chunks].cpu().numpy()
        assert np.array_equal(ca, cb), (name, trial)
        oa, ob = a.output(), b.output()
        for c in np.nonzero(sb == 0)[0]:
            lo, n = int(enc.table["out_off"][c]), int(enc.table["n"][c])
            assert np.array_equal(oa[lo:lo + n], ob[lo:lo + n]), (name, trial, c)


def raw_chunks_longer_than_the_levels():
    """Codec-level (raw) SIMD-BP128 chunks may hold more than 65,536 integers, i.e. more
    blocks than levels x segment size: the last level takes the remainder.  Against the
    one-warp kernel and the input (called inside the forced subprocess)."""
    codec = P.make_codec("simdbp128")
    rng = np.random.default_rng(31)
    lens = np.array([128 * 3000, 128 * 513, 65536, 128 * 1025, 128, 128 * 7], np.uint32)
    offs = np.concatenate([[0], np.cumsum(lens, dtype=np.uint64)[:-1]]).astype(np.uint64)
    flat = rng.integers(0, 1 << 13, size=int(lens.sum()), dtype=np.uint32)
    flat[::977] = rng.integers(0, 2**32, size=len(flat[::977]), dtype=np.uint64).astype(np.uint32)
    enc = H.encode_chunks(codec, flat, offs, lens, raw=True)
    a = P.DeviceBatch(codec, enc, raw=True)
    b = P.DeviceBatch(codec, enc, raw=True, indexed=False)
    assert a.workspace is not None
    a.decode()
    b.decode()
    a.check()
    b.check()
    assert np.array_equal(a.output(), flat) and np.array_equal(b.output(), flat)
    assert np.array_equal(a.consumed[:len(lens)].cpu().numpy(), b.consumed[:len(lens)].cpu().numpy())


@pytest.mark.parametrize("segs", [2, 4, 8, 32])
def test_relay_kernel_parity_suite(cuda, segs):
    _run({"IZG_RELAY": "1", "IZG_SPLIT": "0", "IZG_RELAY_SEGS": str(segs)},
         _SCRIPT.format(root=ROOT))


def test_relay_kernel_config_shapes(cuda, ref):
    _run({"IZG_RELAY": "1", "IZG_SPLIT": "0"},
         f"import sys; sys.path.insert(0, {ROOT!r}); from tests.config_cases import main; main()")


def test_relay_default_routing_ragged_batch(cuda):
    """4,096 chunks (C3's count) of ragged lengths with some corrupted: the
    batch takes the relay by default (workspace given) and must equal the
    one-warp kernel chunk for chunk, repeatedly (tasks of different chunks
    and levels interleave differently every launch)."""
    from paper_1209_2137_b200 import _native as N

    codec = P.make_codec("simdbp128-s4")
    assert N.lib().izg_decode_workspace_size(codec.codec, 4096) >= 4096 * 64
    rng = np.random.default_rng(99)
    count = 4096
    counts = rng.choice([65536, 65536, 65536, 40000, 8192 + 77, 2048, 300, 1], size=count)
    counts = counts.astype(np.uint32)
    offs = np.concatenate([[0], np.cumsum(counts, dtype=np.uint64)[:-1]]).astype(np.uint64)
    total = int(counts.sum())
    gaps = rng.integers(0, 1 << 11, size=total, dtype=np.uint32)
    flat = np.empty(total, np.uint32)
    for o, n in zip(offs, counts):  # sorted per array, wrapping mod 2^32 is fine for D4
        flat[int(o):int(o) + int(n)] = np.cumsum(gaps[int(o):int(o) + int(n)], dtype=np.uint32)
    enc = H.encode_chunks(codec, flat, offs, counts, allow_wrap=True)
    w = enc.words.copy()
    hit = rng.choice(count, size=64, replace=False)
    for c in hit:
        off, nw = int(enc.table["word_off"][c]), int(enc.table["n_words"][c])
        w[off + int(rng.integers(0, nw))] ^= np.uint32(1) << np.uint32(rng.integers(0, 32))
    bad = Encoded(w, enc.table)
    a = P.DeviceBatch(codec, bad, relay_long_only=False)
    b = P.DeviceBatch(codec, bad, indexed=False)
    assert a.workspace is not None
    b.decode()
    sb, ob = b.statuses(), b.output()
    assert (sb == 0).sum() >= count - 64
    clean = np.ones(count, bool)
    clean[hit] = False  # a flipped payload bit may still decode, to other values
    assert (sb[clean] == 0).all()
    cm = np.repeat(clean, counts)
    assert np.array_equal(ob[cm], flat[cm])
    good = np.repeat(sb == 0, counts)
    for rep in range(3):
        a.out.fill_(0)
        a.decode()
        assert np.array_equal(a.statuses(), sb), rep
        assert np.array_equal(a.output()[good], ob[good]), rep
        assert np.array_equal(a.consumed[:count].cpu().numpy(), b.consumed[:count].cpu().numpy())


@pytest.mark.parametrize("env", [{}, {"IZG_RELAY": "1", "IZG_SPLIT": "0", "IZG_CTA": "0"}])
def test_relay_randomized_stress_short(cuda, env):
    """tools/relay_stress.py for 15 s: random batch sizes, ragged lengths, delta modes and
    the raw mode, bit flips and truncated payloads, against the one-warp kernel (a
    10-minute run: profiles/r02_relay_stress.log, 1.06 M chunks)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "relay_stress.py"), "15", "7"],
                       cwd=ROOT, env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().startswith("ok:"), r.stdout[-1000:] + r.stderr[-3000:]


@pytest.mark.parametrize("n", [1, 100, 1000, 8192 + 5])
def test_relay_default_routing_short_chunks(cuda, n):
    """Batches of short chunks in the relay's default range: every chunk has one segment
    (or two), the warps leave at the first task of a level no chunk reaches."""
    codec = P.make_codec("simdbp128-s4")
    count = 5000
    rng = np.random.default_rng(n)
    flat = np.cumsum(rng.integers(0, 64, size=(count, n), dtype=np.uint32), axis=1,
                     dtype=np.uint32).reshape(-1)
    offs = np.arange(count, dtype=np.uint64) * n
    enc = H.encode_chunks(codec, flat, offs, np.full(count, n, np.uint32))
    assert P.DeviceBatch(codec, enc).workspace is None  # short chunks: one warp per chunk
    b = P.DeviceBatch(codec, enc, relay_long_only=False)
    assert b.workspace is not None
    for _ in range(3):
        b.out.fill_(0)
        b.decode()
        b.check()
        assert np.array_equal(b.output(), flat)
