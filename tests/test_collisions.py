"""Exception collisions and extremes on hand-built pages (tests/page_builder):
duplicate exception positions (they OR together, codec_patched.cpp:401-404),
255 exceptions in one block, 32-bit and 1-bit exception widths, for the
vertical (simdfastpfor) and scalar (fastpfor) layouts.  The builder and the
oracle are pinned to the reference here on CPU; the GPU test holds the
kernels to the same bytes."""
import numpy as np
import pytest

import paper_1209_2137_b200 as P
from tests.page_builder import build_fastpfor_page


def blocks_for(rng, nblocks=12):
    out = []
    for k in range(nblocks):
        kind = k % 6
        if kind == 0:    # 255 exceptions with many duplicate positions
            b, mb, c = 7, 19, 255
        elif kind == 1:  # b = 0: every value is an exception of width 32
            b, mb, c = 0, 32, 128
        elif kind == 2:  # 1-bit exceptions on 31-bit values
            b, mb, c = 31, 32, 40
        elif kind == 3:  # no exceptions
            b, mb, c = int(rng.integers(0, 33)), None, 0
        elif kind == 4:  # a single exception, duplicated
            b, mb, c = 3, 9, 2
        else:
            b = int(rng.integers(0, 30))
            mb = int(rng.integers(b + 1, 33))
            c = int(rng.integers(1, 60))
        mb = b if mb is None else mb
        low = rng.integers(0, 2**32, size=128, dtype=np.uint64)
        if kind == 4:
            pos = [77, 77]
        else:
            pos = sorted(int(x) for x in rng.integers(0, 128, size=c))
        highs = [int(x) for x in rng.integers(0, 2**32, size=c, dtype=np.uint64)]
        out.append((low, b, mb, pos, highs))
    return out


@pytest.mark.parametrize("vertical", [True, False])
def test_builder_and_oracle_match_reference(oracle, ref, vertical):
    name = "simdfastpfor" if vertical else "fastpfor"
    for seed in range(4):
        page, expect = build_fastpfor_page(blocks_for(np.random.default_rng(seed)), vertical)
        got, used = ref.decode_deltas(name, page, len(expect))
        assert np.array_equal(got, expect) and used == len(page)
        st, oout, oused = oracle.decode_deltas(name, page, len(expect))
        assert st == 0 and np.array_equal(oout, expect) and oused == len(page)


@pytest.mark.gpu
@pytest.mark.parametrize("vertical", [True, False])
def test_collisions_on_gpu(cuda, oracle, vertical):
    name = "simdfastpfor" if vertical else "fastpfor"
    codec = P.make_codec(name)
    pages, expects = [], []
    for seed in range(12):
        page, expect = build_fastpfor_page(blocks_for(np.random.default_rng(100 + seed)),
                                           vertical)
        pages.append(page)
        expects.append(expect)
    enc = P.layout(codec, pages, [len(e) for e in expects])
    flat = np.concatenate(expects)
    for indexed in (False, True):
        b = P.DeviceBatch(codec, enc, raw=True, indexed=indexed)
        b.decode()
        assert not b.statuses().any()
        assert np.array_equal(b.output(), flat)
        assert list(b.consumed[:b.n_chunks].cpu().numpy()) == [len(p) for p in pages]
    # and through the array pipeline with D4 (decode_array semantics)
    got, st = P.decode_array(codec, enc, raw=True, return_status=True)
    assert not st.any() and np.array_equal(got, flat)
