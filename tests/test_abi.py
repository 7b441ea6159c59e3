"""The C ABI library: loads, exports every symbol include/intzip_b200.h
declares, host-side logic behaves, and compute entry points refuse to run
without a B200 (there is no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1209_2137_b200 as P
from paper_1209_2137_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(header).read()
    return sorted(set(re.findall(r"^\s*[A-Za-z_][\w\s\*]*?\b(izg_\w+)\s*\(", text, re.M)))


def test_exports_every_declared_symbol(native):
    lib = C.CDLL(N.LIB_PATH)
    names = declared(os.path.join(ROOT, "include", "intzip_b200.h"))
    assert set(N.ABI_SYMBOLS) <= set(names)
    for name in names:
        assert hasattr(lib, name), name


def test_product_library_exports_only_the_abi(native):
    """The decoder .so exports the C ABI and nothing from the bench/test
    harness (generators, host encoder: harness/libizh.so)."""
    import shutil
    import subprocess

    nm = shutil.which("nm")
    if not nm:
        pytest.skip("nm not available")
    out = subprocess.run([nm, "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    ours = {s for s in exported if s.startswith(("izg_", "izh_", "izr_"))}
    names = set(declared(os.path.join(ROOT, "include", "intzip_b200.h")))
    assert ours <= names, sorted(ours - names)
    assert not any(s.startswith("izh_") for s in exported)


def test_harness_placement_equals_layout_contract():
    import harness as H

    rng = np.random.default_rng(9)
    for name, codec in (("simdbp128-s4", N.SIMDBP128), ("simdfastpfor-s4", N.SIMDFASTPFOR)):
        lens = rng.integers(1, 70000, size=40).astype(np.uint64)
        vals = np.sort(rng.integers(0, 2**31, size=int(lens.sum()), dtype=np.uint64)).astype(np.uint32)
        offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
        counts = np.minimum(lens, 65536).astype(np.uint32)
        enc = H.encode_chunks(name, vals, offs, counts)
        sizes = enc.table["n_words"].copy()
        woff = np.empty(len(sizes), np.uint64)
        total = N.lib().izg_layout_chunks(codec, N.ptr(sizes), len(sizes), N.ptr(woff))
        assert np.array_equal(woff, enc.table["word_off"]) and total == len(enc.words)


def test_library_targets_sm100a(native):
    """The fatbinary carries sm_100a SASS (cuobjdump lists the ELF arch)."""
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_codec_registry():
    """make_codec (codec.cpp:99-109) for the hot-path names."""
    assert P.make_codec("simdbp128").delta == N.DELTA_D1
    assert P.make_codec("simdbp128-s4").delta == N.DELTA_D4
    assert P.make_codec("simdfastpfor").codec == N.SIMDFASTPFOR
    assert P.make_codec("simdfastpfor-s4").delta == N.DELTA_D4
    assert P.make_codec("simdbp128-d2").delta == N.DELTA_D2
    assert P.make_codec("simdfastpfor-dm").delta == N.DELTA_DM
    # the scalar-group codecs of SURVEY.md §8 f3 (decode only)
    assert P.make_codec("bp32").codec == 2 and P.make_codec("fastpfor-s4").codec == 3
    assert P.make_codec("simplepfor").codec == 4
    for bad in ("lz77", "", "simdbp128-s5", "vbyte", "pfor"):
        with pytest.raises(ValueError):
            P.make_codec(bad)
    assert P.codec_names() == ["simdbp128", "simdbp128-s4", "simdfastpfor", "simdfastpfor-s4"]


def test_status_strings_match_reference_messages():
    assert N.status_string(0) == "ok"
    assert N.status_string(7) == "simdbp128: width byte exceeds 32"
    assert N.status_string(21) == "fastpfor: exception array exhausted"
    with pytest.raises(P.CorruptError):
        P.raise_for_status(16)
    with pytest.raises(ValueError):
        P.raise_for_status(64)


@pytest.mark.parametrize("codec", [N.SIMDBP128, N.SIMDFASTPFOR])
def test_layout_contract(codec):
    rng = np.random.default_rng(codec)
    sizes = rng.integers(0, 5000, size=300).astype(np.uint32)
    offs = np.empty(len(sizes), np.uint64)
    total = N.lib().izg_layout_chunks(codec, N.ptr(sizes), len(sizes), N.ptr(offs))
    phase = 3 if codec == N.SIMDFASTPFOR else 0
    assert np.all(offs % 4 == phase)
    ends = offs + sizes
    assert np.all(offs[1:] >= ends[:-1])  # no overlap
    # the 16-byte-aligned span of every chunk lies inside the allocation
    assert total % 4 == 0 and total >= ((int(ends.max()) + 3) // 4) * 4
    assert np.all(offs - offs % 4 >= 0)


def test_compute_entry_points_refuse_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    L = N.lib()
    words = np.zeros(64, np.uint32)
    table = np.zeros(1, N.CHUNK_DTYPE)
    out = np.zeros(128, np.uint32)
    st = np.zeros(1, np.int32)
    rc = L.izg_decode(0, 2, N.ptr(words), N.ptr(table), 1, N.ptr(out), N.ptr(st), None, None)
    assert rc in (N.ERR_NO_DEVICE, N.ERR_INVALID_ARGUMENT)
    rc = L.izg_decode_host(0, 2, N.ptr(words), 64, N.ptr(table), 1, N.ptr(out), 128, N.ptr(st))
    assert rc == N.ERR_NO_DEVICE
    with pytest.raises(RuntimeError):
        P.decode_array(P.make_codec("simdbp128-s4"), P.Encoded(words, table))


def test_decode_argument_validation():
    L = N.lib()
    assert L.izg_decode(7, 2, None, None, 1, None, None, None, None) == N.ERR_INVALID_ARGUMENT
    assert L.izg_decode(0, 9, None, None, 1, None, None, None, None) == N.ERR_INVALID_ARGUMENT
    assert L.izg_decode(0, 2, None, None, 0, None, None, None, None) == N.SUCCESS


def test_workspace_sizes_by_batch():
    """izg_decode_workspace_size (a host-side function): SIMD-BP128 asks for the
    split kernel's states on small batches, for the relay kernel's 64 bytes per
    chunk (+ the task counter) from 2,432 to 14,208 chunks and for nothing
    elsewhere; SIMD-FastPFOR always asks for at least its page index."""
    env = {k: os.environ.get(k) for k in ("IZG_RELAY", "IZG_SPLIT")}
    if any(v is not None for v in env.values()):
        pytest.skip("forced decode paths in the environment")
    L = N.lib()
    bp, fp = P.make_codec("simdbp128-s4").codec, P.make_codec("simdfastpfor-s4").codec
    assert L.izg_decode_workspace_size(bp, 64) > 0            # split
    assert L.izg_decode_workspace_size(bp, 1024) == 0         # CTA kernel: no workspace
    assert L.izg_decode_workspace_size(bp, 2431) == 0
    for n in (2432, 4096, 14208):
        assert L.izg_decode_workspace_size(bp, n) == 64 * n + 64
    assert L.izg_decode_workspace_size(bp, 14209) == 0
    for n in (64, 4096, 65536):
        assert L.izg_decode_workspace_size(fp, n) >= L.izg_decode_index_workspace_size(fp, n) > 0


def test_checksum_host_matches_numpy():
    import harness as H
    from paper_1209_2137_b200.device import host_checksum

    v = np.random.default_rng(1).integers(0, 2**32, size=100003, dtype=np.uint64).astype(np.uint32)
    assert H.checksum_host(v, 17, threads=4) == host_checksum(v, 17)
