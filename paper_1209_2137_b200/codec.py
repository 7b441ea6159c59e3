"""Python mirror of the reference codec interface for the hot path.

Mirrors ``intzip::Codec`` / ``make_codec`` / ``encode_array`` /
``decode_array`` (/root/reference/proj/core/include/intzip/codec.h:23-77) so
parity tests read like the reference's own tests.  Decoding always runs the
fused sm_100a kernel through the C ABI (include/intzip_b200.h); encoding runs
the host encoder mirror of libintzip_b200.  Errors: ``CorruptError`` where the
reference throws ``intzip::CorruptError`` (errors.h:8-14), ``ValueError``
where it throws ``std::invalid_argument``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._native import CHUNK_DTYPE

CHUNK_SIZE = 1 << 16  # kChunkSize (codec.h:17)
DELTA_NAMES = {N.DELTA_NONE: "none", N.DELTA_D1: "scalar", N.DELTA_D4: "stride4",
               N.DELTA_D2: "stride2(ext)", N.DELTA_DM: "max4(ext)"}


SPLIT_STALL = 38  # IZG_E_SPLIT_STALL


class CorruptError(RuntimeError):
    """intzip::CorruptError (errors.h:8-14): malformed compressed input."""

    def __init__(self, status: int, chunk: int | None = None):
        self.status = int(status)
        self.chunk = chunk
        where = "" if chunk is None else f" (chunk {chunk})"
        super().__init__(N.status_string(status) + where)


def raise_for_status(status: int, chunk: int | None = None) -> None:
    if status == 0:
        return
    if status >= 64:  # std::invalid_argument sites
        raise ValueError(N.status_string(status))
    if status == SPLIT_STALL:  # internal error of the split decode, not the input
        raise RuntimeError(N.status_string(status))
    raise CorruptError(status, chunk)


@dataclass(frozen=True)
class Codec:
    """intzip::Codec (codec.h:23-52) for simdbp128[-s4] / simdfastpfor[-s4]."""
    name: str
    codec: int
    delta: int
    block_multiple: int = 128  # codec_binpack.cpp:64-66, codec_patched.cpp:216-217

    @property
    def delta_mode(self) -> str:
        return DELTA_NAMES[self.delta]


def make_codec(name: str) -> Codec:
    """make_codec (codec.cpp:99-109); unknown names raise ValueError."""
    c, d = C.c_int(), C.c_int()
    rc = N.lib().izg_parse_codec_name(name.encode(), C.byref(c), C.byref(d))
    if rc != N.SUCCESS:
        raise ValueError(f"unknown codec: {name}")
    return Codec(name, c.value, d.value)


def codec_names() -> list[str]:
    """The hot-path subset of codec_names() (codec.cpp:111-119)."""
    return ["simdbp128", "simdbp128-s4", "simdfastpfor", "simdfastpfor-s4"]


@dataclass
class Encoded:
    """Chunks of one or more arrays laid out for the device (izg_layout_chunks)."""
    words: np.ndarray  # uint32, 16-byte-aligned placement contract
    table: np.ndarray  # CHUNK_DTYPE

    @property
    def n_out(self) -> int:
        if len(self.table) == 0:
            return 0
        return int((self.table["out_off"] + self.table["n"]).max())

    @property
    def payload_words(self) -> int:
        return int(self.table["n_words"].sum())


def encode_array(codec: Codec, values, *, allow_wrap: bool = False, device=None) -> Encoded:
    """encode_array (codec.cpp:14-37) on the GPU encoder (izg_encode): chunks
    of 2^16, delta, core, VByte tail.  Raises ValueError where the reference
    throws std::invalid_argument (a decreasing input, delta.cpp:13)."""
    from .device import encode_on_device

    values = np.ascontiguousarray(values, dtype=np.uint32)
    n = len(values)
    offs = np.arange(0, n, CHUNK_SIZE, dtype=np.uint64)
    counts = np.minimum(CHUNK_SIZE, n - offs).astype(np.uint32)
    enc, status = encode_on_device(codec, values, offs, counts, allow_wrap=allow_wrap,
                                   device=device)
    bad = np.nonzero(status)[0]
    if len(bad):
        raise_for_status(int(status[bad[0]]), int(bad[0]))
    return enc


def layout(codec: Codec, payloads: list[np.ndarray], counts, out_offs=None) -> Encoded:
    """Place existing chunk payloads (e.g. from the CPU reference) for the device."""
    sizes = np.array([len(p) for p in payloads], dtype=np.uint32)
    offs = np.empty(len(payloads), dtype=np.uint64)
    total = N.lib().izg_layout_chunks(codec.codec, N.ptr(sizes), len(payloads), N.ptr(offs))
    words = np.zeros(total, dtype=np.uint32)
    for p, o in zip(payloads, offs):
        words[int(o):int(o) + len(p)] = p
    table = np.empty(len(payloads), dtype=CHUNK_DTYPE)
    table["word_off"] = offs
    table["n_words"] = sizes
    table["n"] = np.asarray(counts, dtype=np.uint32)
    if out_offs is None:
        out_offs = np.concatenate([[0], np.cumsum(table["n"].astype(np.uint64))[:-1]])
    table["out_off"] = out_offs
    return Encoded(words, table)


def decode_array(codec: Codec, enc: Encoded, *, raw: bool = False,
                 return_status: bool = False):
    """decode_array (codec.cpp:39-76) through the GPU, host buffers in and out.

    Raises CorruptError / ValueError with the first failing chunk's status
    (the reference throws at the first failing chunk) unless return_status.
    """
    L = N.lib()
    n_out = enc.n_out
    out = np.zeros(max(n_out, 1), dtype=np.uint32)
    status = np.zeros(max(len(enc.table), 1), dtype=np.int32)
    delta = N.DELTA_NONE if raw else codec.delta
    rc = L.izg_decode_host(codec.codec, delta, N.ptr(enc.words), len(enc.words),
                           N.ptr(enc.table), len(enc.table), N.ptr(out), len(out),
                           N.ptr(status))
    if rc not in (N.SUCCESS, N.ERR_CORRUPT):
        raise RuntimeError(f"izg_decode_host failed: {rc}")
    status = status[:len(enc.table)]
    if return_status:
        return out[:n_out], status
    bad = np.nonzero(status)[0]
    if len(bad):
        raise_for_status(int(status[bad[0]]), int(bad[0]))
    return out[:n_out]
