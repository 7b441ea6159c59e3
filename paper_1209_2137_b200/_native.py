"""ctypes binding of libintzip_b200.so (include/intzip_b200.h).

The library must exist: there is no CPU fallback.  Build it with
``python -m paper_1209_2137_b200.build`` (or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# IZG_LIB_PATH: developer A/B runs of alternative builds (tools/); the default
# is the in-tree build.
LIB_PATH = os.environ.get("IZG_LIB_PATH") or os.path.join(_HERE, "_lib", "libintzip_b200.so")

# izg_chunk (include/intzip_b200.h): 24 bytes, naturally aligned.
CHUNK_DTYPE = np.dtype([("word_off", "<u8"), ("n_words", "<u4"), ("n", "<u4"),
                        ("out_off", "<u8")])
assert CHUNK_DTYPE.itemsize == 24

SIMDBP128, SIMDFASTPFOR = 0, 1
DELTA_NONE, DELTA_D1, DELTA_D4, DELTA_D2, DELTA_DM = 0, 1, 2, 3, 4

SUCCESS = 0
ERR_INVALID_ARGUMENT = -1
ERR_CUDA = -2
ERR_NO_DEVICE = -3
ERR_CORRUPT = -4
ERR_UNKNOWN_CODEC = -5

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def lib() -> C.CDLL:
    """Load the native library (raises loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} not found: build it with `python -m paper_1209_2137_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    u32p, u64p, i32p = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_int32)
    vp = C.c_void_p
    L.izg_status_string.restype = C.c_char_p
    L.izg_status_string.argtypes = [C.c_int32]
    L.izg_parse_codec_name.restype = C.c_int
    L.izg_parse_codec_name.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.izg_layout_chunks.restype = C.c_uint64
    L.izg_layout_chunks.argtypes = [C.c_int, vp, C.c_uint32, vp]
    L.izg_decode.restype = C.c_int
    L.izg_decode.argtypes = [C.c_int, C.c_int, vp, vp, C.c_uint32, vp, vp, vp, vp]
    L.izg_decode_ws.restype = C.c_int
    L.izg_decode_ws.argtypes = [C.c_int, C.c_int, vp, vp, C.c_uint32, vp, vp, vp, vp,
                                C.c_uint64, vp]
    L.izg_decode_ws_phase.restype = C.c_int
    L.izg_decode_ws_phase.argtypes = [C.c_int, C.c_int, vp, vp, C.c_uint32, vp, vp, vp, vp,
                                      C.c_uint64, C.c_int, vp]
    L.izg_decode_workspace_size.restype = C.c_uint64
    L.izg_decode_workspace_size.argtypes = [C.c_int, C.c_uint32]
    L.izg_decode_index_workspace_size.restype = C.c_uint64
    L.izg_decode_index_workspace_size.argtypes = [C.c_int, C.c_uint32]
    L.izg_container_scan.restype = C.c_int
    L.izg_container_scan.argtypes = [vp, C.c_uint64, C.c_int, vp, vp]
    L.izg_container_index.restype = C.c_int
    L.izg_container_index.argtypes = [vp, C.c_uint64, vp, vp, vp]
    L.izg_container_decode_host.restype = C.c_int
    L.izg_container_decode_host.argtypes = [vp, C.c_uint64, vp, C.c_uint64, vp, vp]
    L.izg_intersect_workspace_size.restype = C.c_uint64
    L.izg_intersect_workspace_size.argtypes = [C.c_uint64, C.c_uint64]
    L.izg_intersect_sorted.restype = C.c_int
    L.izg_intersect_sorted.argtypes = [vp, C.c_uint64, vp, C.c_uint64, vp, vp, vp, C.c_uint64,
                                       vp]
    L.izg_decode_intersect_workspace_size.restype = C.c_uint64
    L.izg_decode_intersect_workspace_size.argtypes = [C.c_uint64]
    L.izg_decode_intersect.restype = C.c_int
    L.izg_decode_intersect.argtypes = [C.c_int, C.c_int, vp, vp, C.c_uint32, vp, C.c_uint64, vp,
                                       vp, vp, vp, C.c_uint64, vp]
    L.izg_checksum.restype = C.c_int
    L.izg_checksum.argtypes = [vp, C.c_uint64, vp, vp]
    L.izg_decode_host.restype = C.c_int
    L.izg_decode_host.argtypes = [C.c_int, C.c_int, vp, C.c_uint64, vp, C.c_uint32, vp,
                                  C.c_uint64, vp]
    L.izg_release_host_scratch.restype = None
    L.izg_release_host_scratch.argtypes = []
    L.izg_encode.restype = C.c_int
    L.izg_encode.argtypes = [C.c_int, C.c_int, vp, vp, C.c_uint32, vp, vp, C.c_int, vp]
    L.izg_encode_bound.restype = C.c_uint64
    L.izg_encode_bound.argtypes = [C.c_int, C.c_uint32]
    _lib = L
    return L


# Symbols include/intzip_b200.h declares (checked by the CPU test suite).
ABI_SYMBOLS = ("izg_status_string", "izg_parse_codec_name", "izg_layout_chunks",
               "izg_decode", "izg_decode_ws", "izg_decode_ws_phase", "izg_decode_workspace_size",
               "izg_decode_index_workspace_size", "izg_checksum", "izg_decode_host", "izg_release_host_scratch",
               "izg_encode", "izg_encode_bound", "izg_container_scan", "izg_container_index",
               "izg_container_decode_host", "izg_intersect_workspace_size",
               "izg_intersect_sorted", "izg_decode_intersect_workspace_size",
               "izg_decode_intersect")


def ptr(a) -> int:
    """Address of a numpy array or torch tensor."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def status_string(s: int) -> str:
    return lib().izg_status_string(int(s)).decode()
