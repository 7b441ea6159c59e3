"""INTZPK01 container ingest (the reference's container.h:14-26 format).

Mirrors intzip::container_read_encoded / container_read_raw
(container.cpp:93-169) over an in-memory buffer, through the C ABI
(izg_container_scan / izg_container_index): the container is validated with
the reference's statuses and its chunks are indexed in place, so the body is
handed to the device as one block.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._native import CHUNK_DTYPE
from .codec import Codec, CorruptError, Encoded, make_codec, raise_for_status


class ContainerInfo(C.Structure):
    _fields_ = [("codec_name", C.c_char * 260), ("n_arrays", C.c_uint32),
                ("n_chunks", C.c_uint32), ("n_values", C.c_uint64),
                ("body_offset", C.c_uint64), ("body_words", C.c_uint64)]


def _buffer(data) -> np.ndarray:
    if isinstance(data, np.ndarray):
        return np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    return np.frombuffer(bytes(data), dtype=np.uint8)


def scan_container(data, raw: bool = False) -> ContainerInfo:
    """Validate a container; raises CorruptError with the reference's status."""
    buf = _buffer(data)
    info = ContainerInfo()
    st = C.c_int32(0)
    rc = N.lib().izg_container_scan(N.ptr(buf) if len(buf) else None, len(buf), int(raw),
                                    C.byref(info), C.byref(st))
    if rc == N.ERR_CORRUPT:
        raise CorruptError(st.value)
    if rc != N.SUCCESS:
        raise RuntimeError(f"izg_container_scan failed: {rc}")
    return info


@dataclass
class Container:
    """container_read_encoded's EncodedContainer, laid out for the device."""
    codec_name: str
    encoded: Encoded          # body words (in place) + chunk table
    array_chunk0: np.ndarray  # n_arrays + 1 first-chunk indices
    array_offsets: np.ndarray  # n_arrays + 1 output offsets

    @property
    def codec(self) -> Codec:
        return make_codec(self.codec_name)


def read_container(data) -> Container:
    buf = _buffer(data)
    info = scan_container(buf)
    table = np.zeros(info.n_chunks, dtype=CHUNK_DTYPE)
    chunk0 = np.zeros(info.n_arrays + 1, dtype=np.uint32)
    rc = N.lib().izg_container_index(N.ptr(buf), len(buf), C.byref(info),
                                     N.ptr(table) if len(table) else None, N.ptr(chunk0))
    if rc != N.SUCCESS:
        raise RuntimeError(f"izg_container_index failed: {rc}")
    # body words, padded so every chunk's 16-byte span lies inside the buffer
    nb = int(info.body_words)
    words = np.zeros((nb + 3) // 4 * 4 + 4, dtype=np.uint32)
    body = buf[int(info.body_offset):int(info.body_offset) + 4 * nb]
    words.view(np.uint8)[:len(body)] = body
    offs = np.append(table["out_off"], np.uint64(info.n_values))[chunk0.astype(np.int64)]
    return Container(info.codec_name.decode(), Encoded(words, table), chunk0, offs)


def read_raw_container(data) -> list[np.ndarray]:
    """container_read_raw (container.cpp:93-110)."""
    buf = _buffer(data)
    info = scan_container(buf, raw=True)
    table = np.zeros(info.n_arrays, dtype=CHUNK_DTYPE)
    if info.n_arrays:
        N.lib().izg_container_index(N.ptr(buf), len(buf), C.byref(info), N.ptr(table), None)
    base = int(info.body_offset)
    out = []
    for t in table:
        o = base + 4 * int(t["word_off"])
        out.append(buf[o:o + 4 * int(t["n"])].view(np.uint32).copy())
    return out


def decode_container(data) -> tuple[np.ndarray, np.ndarray]:
    """Read + decode an encoded container on the GPU (izg_container_decode_host).

    Returns (values of all arrays back to back, n_arrays + 1 array offsets);
    raises CorruptError (container or first failing chunk) like the reference.
    """
    buf = _buffer(data)
    info = scan_container(buf)
    out = np.zeros(max(int(info.n_values), 1), dtype=np.uint32)
    st = np.zeros(max(int(info.n_chunks), 1), dtype=np.int32)
    ct = C.c_int32(0)
    rc = N.lib().izg_container_decode_host(N.ptr(buf), len(buf), N.ptr(out), len(out),
                                           C.byref(ct), N.ptr(st))
    if rc == N.ERR_UNKNOWN_CODEC:
        raise ValueError(f"unknown codec: {info.codec_name.decode()}")
    if ct.value:
        raise CorruptError(ct.value)
    if rc not in (N.SUCCESS, N.ERR_CORRUPT):
        raise RuntimeError(f"izg_container_decode_host failed: {rc}")
    bad = np.nonzero(st[:info.n_chunks])[0]
    if len(bad):
        raise_for_status(int(st[bad[0]]), int(bad[0]))
    c = read_container(buf)
    return out[:info.n_values], c.array_offsets
