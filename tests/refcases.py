"""The reference's own known-answer tests for the hot path, restated.

Every case cites the reference test it restates (paths under
/root/reference/proj/tests/).  The expected values are the reference's
literals; the tests run them against the oracle, the reference library
compiled from source, the product's host encoder, and (gpu-marked) the fused
CUDA decoder.
"""
from __future__ import annotations

import numpy as np

U32 = np.uint32


def ref_pack_bits(values, b):
    """testutil.h:13-23 — bit i*b+k of a flat bit string."""
    words = np.zeros((len(values) * b + 31) // 32, dtype=np.uint64)
    for i, v in enumerate(values):
        for k in range(b):
            if (int(v) >> k) & 1:
                p = i * b + k
                words[p // 32] |= 1 << (p % 32)
    return words.astype(U32)


def ref_pack_vertical(values, b):
    """testutil.h:38-48 — four round-robin lanes interleaved word by word."""
    out = np.zeros(4 * b, dtype=U32)
    for j in range(4):
        lane = [values[4 * i + j] for i in range(32)]
        packed = ref_pack_bits(lane, b)
        for i in range(b):
            out[4 * i + j] = packed[i]
    return out


def random_block(rng: np.random.Generator, n, b):
    """testutil.h:64-71 (numpy generator instead of mt19937_64)."""
    mask = (1 << b) - 1 if b < 32 else 0xFFFFFFFF
    return (rng.integers(0, 2**32, size=n, dtype=np.uint64) & mask).astype(U32)


# codec_patched_test.cpp:16-25 — the worked block, padded to 128 with 2s.
WORKED_BLOCK = [2, 2, 1, 2, 38, 2, 1, 3, 2, 32, 2, 52, 2, 3, 3, 1]


def worked_page128():
    return np.array(WORKED_BLOCK + [2] * (128 - 16), dtype=U32)


def worked_page_expected_words():
    """codec_patched_test.cpp:274-301 — the 32-word SIMD-FastPFOR golden page
    (fields the reference test pins; words 1..8 are the vertical pack of the
    page at b=2 and words 10..11 the byte array, checked by equality with
    ref_pack_vertical and the byte layout)."""
    page = worked_page128()
    highs = np.zeros(128, dtype=U32)
    highs[:3] = [9, 8, 13]
    return {
        "size": 32,
        0: 9, 9: 6, 12: 1 << 3, 13: 3, 14: 0, 15: 0,
        "packed_1_9": ref_pack_vertical(page & 3, 2),
        "highs_16_32": ref_pack_vertical(highs, 4),
        # byte array: b=2, maxbits=6, c=3, positions 4, 9, 11; then 127 blocks... only one block
        "byte_array": [2, 6, 3, 4, 9, 11],
    }


# codec_patched_test.cpp:53-61 — cost goldens of the worked block.
WORKED_COSTS = {1: 185, 2: 68, 6: 96}
WORKED_CHOICE = (2, 6)

# codec_basic_test.cpp:16-32 — VByte goldens.
VBYTE_GOLDENS = [(0, [0x80]), (127, [0xFF]), (128, [0x00, 0x81]), (200, [0x48, 0x81]),
                 (0xFFFFFFFF, [0x7F, 0x7F, 0x7F, 0x7F, 0x8F])]
# codec_basic_test.cpp:58-77 — decode errors (bytes, count, izg status).
VBYTE_ERRORS = [([0x01], 1, 3),                                   # truncated
                ([0x01, 0x01, 0x01, 0x01, 0x01, 0x81], 1, 5),     # > 5 bytes
                ([0x00, 0x00, 0x00, 0x00, 0x80 | 0x10], 1, 4)]    # > 32 bits

# delta_test.cpp:14-18, 43-49
D1_EXAMPLE = ([1, 3, 9], [1, 4, 13])
D4_EXAMPLE = ([1, 2, 3, 4, 10, 12, 13, 14], [1, 2, 3, 4, 9, 10, 10, 10])
