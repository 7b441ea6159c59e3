"""B200-native fused SIMD-BP128 / SIMD-FastPFOR decoder (arXiv 1209.2137 hot path).

The product is libintzip_b200.so (paper_1209_2137_b200/_lib), whose C ABI is
include/intzip_b200.h; this package is its Python face (ctypes).
"""
from . import _native
from .codec import (CHUNK_SIZE, Codec, CorruptError, Encoded, codec_names, decode_array,
                    encode_array, layout, make_codec, raise_for_status)
from .container import (Container, decode_container, read_container, read_raw_container,
                        scan_container)
from .device import DeviceBatch, decode_intersect_device, intersect, intersect_device

__all__ = ["CHUNK_SIZE", "Codec", "Container", "CorruptError", "DeviceBatch", "Encoded",
           "codec_names", "decode_container", "decode_intersect_device", "intersect", "intersect_device", "read_container", "read_raw_container",
           "scan_container",
           "decode_array", "encode_array", "layout",
           "make_codec", "raise_for_status", "_native"]
