"""Bench/test harness: seeded BASELINE.json inputs and a host encoder.

NOT the product.  ``libizh.so`` (harness/csrc, built with g++) holds the
synthetic-input generators (``gen_arrays``), a host checksum and a host
encoder for the hot-path codecs (``encode_chunks`` / ``encode_array``, word
for word with the reference encoder — tests/test_oracle_vs_ref.py).  The
decoder library ``paper_1209_2137_b200/_lib/libintzip_b200.so`` neither
contains nor links any of it.  This module imports nothing from the product
package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "_build", "libizh.so")
SOURCES = ["datagen.cpp", "host_encode.cpp"]

CHUNK_SIZE = 1 << 16
# izg_chunk (include/intzip_b200.h)
CHUNK_DTYPE = np.dtype([("word_off", "<u8"), ("n_words", "<u4"), ("n", "<u4"),
                        ("out_off", "<u8")])
# codec / delta ids of include/intzip_b200.h
CODEC_IDS = {"simdbp128": 0, "simdfastpfor": 1}
DELTA_IDS = {"": 1, "-s4": 2, "-d2": 3, "-dm": 4}
MODELS = {"uniform": 0, "cluster": 1, "geometric": 2, "raw": 3}

_lib = None


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))]
    deps.append(os.path.join(ROOT, "include", "intzip_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False) -> str:
    if not force and not _stale():
        return LIB_PATH
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    tmp = LIB_PATH + ".tmp"
    cmd = ["g++", "-std=c++17", "-O3", "-fPIC", "-shared", "-pthread", "-o", tmp,
           *[os.path.join(HERE, "csrc", s) for s in SOURCES]]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.izh_gen_arrays.restype = C.c_int
    L.izh_gen_arrays.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                 C.c_uint64, C.c_uint32, C.c_int, vp, vp]
    L.izh_array_widths.restype = C.c_int
    L.izh_array_widths.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int, vp]
    L.izh_checksum_host.restype = C.c_int
    L.izh_checksum_host.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_int, vp]
    L.izh_encode_batch.restype = vp
    L.izh_encode_batch.argtypes = [C.c_int, C.c_int, vp, vp, vp, C.c_uint32, C.c_int, C.c_int,
                                   C.POINTER(C.c_int)]
    L.izh_encoded_words.restype = C.c_uint64
    L.izh_encoded_words.argtypes = [vp]
    L.izh_encoded_copy.restype = C.c_int
    L.izh_encoded_copy.argtypes = [vp, vp, vp, C.c_int]
    L.izh_encoded_free.restype = None
    L.izh_encoded_free.argtypes = [vp]
    _lib = L
    return L


def _ptr(a) -> int:
    return a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr()


def threads_default() -> int:
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    return max(1, min(64, n))


@dataclass
class Encoded:
    """Chunks of one or more arrays placed for the device (izg_layout_chunks
    placement); the product's ``Encoded`` has the same two fields."""
    words: np.ndarray  # uint32
    table: np.ndarray  # CHUNK_DTYPE

    @property
    def n_out(self) -> int:
        if len(self.table) == 0:
            return 0
        return int((self.table["out_off"] + self.table["n"]).max())

    @property
    def payload_words(self) -> int:
        return int(self.table["n_words"].sum())


def parse_name(name: str) -> tuple[int, int]:
    """(codec id, delta id) of a hot-path codec name (simdbp128[-s4|-d2|-dm], ...)."""
    for base, cid in CODEC_IDS.items():
        if name.startswith(base) and name[len(base):] in DELTA_IDS:
            return cid, DELTA_IDS[name[len(base):]]
    raise ValueError(f"harness encoder: unsupported codec {name}")


def gen_arrays(model: str, count: int, n: int, d, seed: int, *, rate_ppm: int = 0,
               threads: int | None = None, out: np.ndarray | None = None):
    """Seeded synthetic arrays; returns (values[count, n], d[count])."""
    d_lo, d_hi = (d, d) if np.isscalar(d) else d
    if out is None:
        out = np.empty((count, n), dtype=np.uint32)
    dd = np.empty(count, dtype=np.uint32)
    rc = lib().izh_gen_arrays(MODELS[model], count, n, d_lo, d_hi, seed, rate_ppm,
                              threads or threads_default(), _ptr(out), _ptr(dd))
    if rc != 0:
        raise ValueError("gen_arrays: bad arguments")
    return out, dd


def array_widths(count: int, d, seed: int, threads: int | None = None) -> np.ndarray:
    """Per-array d of gen_arrays(…, count, n, d, seed) without generating."""
    d_lo, d_hi = (d, d) if np.isscalar(d) else d
    out = np.empty(count, dtype=np.uint32)
    if lib().izh_array_widths(count, d_lo, d_hi, seed, threads or threads_default(), _ptr(out)):
        raise ValueError("array_widths: bad arguments")
    return out


def checksum_host(v: np.ndarray, base: int = 0, threads: int | None = None) -> tuple[int, int]:
    out = np.zeros(2, dtype=np.uint64)
    lib().izh_checksum_host(_ptr(v), v.size, base, threads or threads_default(), _ptr(out))
    return int(out[0]), int(out[1])


def encode_chunks(codec, values: np.ndarray, value_off, counts, *, allow_wrap: bool = False,
                  raw: bool = False, threads: int | None = None) -> Encoded:
    """Host-encode independent chunks values[value_off[i] : +counts[i]].

    ``codec``: a name, or any object with ``.name`` (e.g. the product's Codec).
    raw=True encodes deltas as-is (Codec::encode_deltas, codec.h:31-34);
    allow_wrap=True takes differences mod 2^32.
    """
    cid, did = parse_name(codec if isinstance(codec, str) else codec.name)
    L = lib()
    values = np.ascontiguousarray(values, dtype=np.uint32)
    value_off = np.ascontiguousarray(value_off, dtype=np.uint64)
    counts = np.ascontiguousarray(counts, dtype=np.uint32)
    st = C.c_int()
    h = L.izh_encode_batch(cid, 0 if raw else did, _ptr(values), _ptr(value_off), _ptr(counts),
                           len(counts), int(allow_wrap), threads or threads_default(),
                           C.byref(st))
    if not h:
        raise ValueError("encode: invalid input (decreasing values or bad counts)")
    try:
        nw = L.izh_encoded_words(h)
        words = np.empty(nw, dtype=np.uint32)
        table = np.empty(len(counts), dtype=CHUNK_DTYPE)
        L.izh_encoded_copy(h, _ptr(words), _ptr(table), threads or threads_default())
    finally:
        L.izh_encoded_free(h)
    return Encoded(words, table)


def encode_array(codec, values, *, allow_wrap: bool = False) -> Encoded:
    """encode_array (codec.cpp:14-37): chunks of 2^16, delta, core, VByte tail."""
    values = np.ascontiguousarray(values, dtype=np.uint32)
    n = len(values)
    offs = np.arange(0, n, CHUNK_SIZE, dtype=np.uint64)
    counts = np.minimum(CHUNK_SIZE, n - offs).astype(np.uint32)
    return encode_chunks(codec, values, offs, counts, allow_wrap=allow_wrap)
