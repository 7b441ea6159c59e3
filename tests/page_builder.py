"""Hand-built SIMD-FastPFOR / FastPFOR pages (test infrastructure).

The reference encoder never emits duplicate exception positions or more than
128 exceptions per block, but its decoder accepts both (codec_patched.cpp
:320-330 bound c by the byte array only and check positions < 128; a
duplicate position ORs twice, :401-404).  These builders lay out such pages
exactly as codec_patched.h:59-80 describes, so the GPU decoder can be held to
the reference on them.
"""
from __future__ import annotations

import numpy as np


def _pack_vertical(values, w):
    """bitpack.h:18-23 vertical layout of 128 values at width w (masked)."""
    out = np.zeros(4 * w, dtype=np.uint64)
    for j in range(4):
        lane = [int(v) & ((1 << w) - 1) if w < 32 else int(v) for v in values[j::4]]
        bits = 0
        for i, v in enumerate(lane):
            bits |= v << (i * w)
        for k in range(w):
            out[4 * k + j] = (bits >> (32 * k)) & 0xFFFFFFFF
    return out.astype(np.uint32)


def _pack_scalar(values, w):
    """bitpack.h:12-16 scalar layout of 32 values at width w (masked)."""
    bits = 0
    for i, v in enumerate(values):
        bits |= (int(v) & ((1 << w) - 1) if w < 32 else int(v)) << (i * w)
    return np.array([(bits >> (32 * k)) & 0xFFFFFFFF for k in range(w)], dtype=np.uint32)


def build_fastpfor_page(blocks, vertical=True):
    """blocks: list of (low[128] uint32, b, maxbits, positions, highs).

    Positions may repeat and len(positions) may exceed 128 (up to 255); the
    block's decoded value at p is low[p] | OR of highs at p shifted by b.
    Returns (payload words, expected decoded deltas)."""
    words = [0]
    ba = bytearray()
    arrays = {w: [] for w in range(1, 33)}
    expect = []
    for low, b, mb, pos, highs in blocks:
        low = np.asarray(low, dtype=np.uint64) & ((1 << b) - 1)
        ba += bytes([b, mb])
        if mb > b:
            assert 0 < len(pos) <= 255 and len(pos) == len(highs)
            ba.append(len(pos))
            ba += bytes(pos)
            for h in highs:
                arrays[mb - b].append(int(h))
        vals = low.copy()
        w = mb - b
        for p, h in zip(pos, highs):
            hm = int(h) & ((1 << w) - 1)
            vals[p] |= (hm << b) & 0xFFFFFFFF
        expect.append(vals.astype(np.uint32))
        if vertical:
            words += list(_pack_vertical(low, b))
        else:
            for g in range(4):
                words += list(_pack_scalar(low[32 * g:32 * g + 32], b))
    words[0] = len(words)
    words.append(len(ba))
    ba += bytes((-len(ba)) % 4)
    words += list(np.frombuffer(bytes(ba), dtype=np.uint32))
    bitset = 0
    for w in range(1, 33):
        if arrays[w]:
            bitset |= 1 << (w - 1)
    words.append(bitset)
    group = 128 if vertical else 32
    for w in range(1, 33):
        hv = arrays[w]
        if not hv:
            continue
        words.append(len(hv))
        if vertical:
            while len(words) % 4:
                words.append(0)
        hv = hv + [0] * ((-len(hv)) % group)
        for g in range(len(hv) // group):
            chunk = hv[group * g:group * (g + 1)]
            words += list(_pack_vertical(chunk, w) if vertical else _pack_scalar(chunk, w))
    return np.array(words, dtype=np.uint32), np.concatenate(expect)
