"""Shared input builders for the parity tests (seeded, deterministic)."""
from __future__ import annotations

import numpy as np

import paper_1209_2137_b200 as P

REF_NAMES = ["simdbp128", "simdbp128-s4", "simdfastpfor", "simdfastpfor-s4"]
EXT_NAMES = ["simdbp128-d2", "simdbp128-dm", "simdfastpfor-d2", "simdfastpfor-dm"]
ALL_NAMES = REF_NAMES + EXT_NAMES
# the same page framework with scalar 32-integer groups
F3_NAMES = ["bp32", "bp32-s4", "fastpfor", "fastpfor-s4", "simplepfor", "simplepfor-s4"]

# Lengths around every boundary of the format: block (128), meta-block
# (2048), chunk (65536), VByte remainder, tiny arrays.
EDGE_LENGTHS = [1, 2, 3, 4, 5, 127, 128, 129, 255, 256, 1000, 2047, 2048, 2049, 4096,
                30000, 65535, 65536, 65537, 140000]


def random_sorted(rng, n, max_delta):
    """testutil.h:52-62: nondecreasing, deltas in [0, max_delta], clamped."""
    d = rng.integers(0, max_delta + 1, size=n, dtype=np.uint64)
    acc = np.minimum(np.cumsum(d), 0xFFFFFFFF)
    return acc.astype(np.uint32)


def assorted_arrays(seed=0):
    rng = np.random.default_rng(seed)
    arrays = [np.zeros(1, np.uint32), np.array([0xFFFFFFFF], np.uint32),
              np.full(300, 77, np.uint32)]  # codec_core_test.cpp:99-115
    for n in EDGE_LENGTHS:
        arrays.append(random_sorted(rng, n, int(rng.choice([1, 50, 1000, 1 << 16, 1 << 24]))))
    # outlier-heavy (patched codec stress, codec_patched_test.cpp:339-358)
    gaps = rng.geometric(1 / 8, size=70000).astype(np.uint64)
    mask = rng.random(70000) < 0.1
    gaps[mask] = rng.integers(1 << 12, 1 << 24, size=int(mask.sum()))
    arrays.append(np.minimum(np.cumsum(gaps), 0xFFFFFFFF).astype(np.uint32))
    # full 32-bit range
    arrays.append(np.sort(rng.integers(0, 2**32, size=5000, dtype=np.uint64)).astype(np.uint32))
    return arrays


def chunks_of(enc: P.Encoded):
    return [(int(t["n"]), enc.words[int(t["word_off"]):int(t["word_off"]) + int(t["n_words"])])
            for t in enc.table]


def misplace(enc: P.Encoded, word_phase: int, out_phase: int, gap: int = 5) -> P.Encoded:
    """Re-place payloads at word offsets = word_phase mod 4 with gaps, and
    outputs at out_phase, to exercise the unaligned paths."""
    chunks = chunks_of(enc)
    total = sum(len(p) + gap + 4 for _, p in chunks) + 16
    words = np.full(total, 0xDEADBEEF, dtype=np.uint32)
    table = np.zeros(len(chunks), dtype=P._native.CHUNK_DTYPE)
    pos, out = 4 + word_phase, out_phase
    for i, (n, p) in enumerate(chunks):
        words[pos:pos + len(p)] = p
        table[i] = (pos, len(p), n, out)
        pos += len(p) + gap
        pos += (word_phase - pos) % 4
        out += n
    return P.Encoded(words, table)
