"""ctypes access to the parity checkers.  TEST INFRASTRUCTURE ONLY.

* ``Oracle``    — oracle/_build/liboracle.so, the C restatement (intzip_oracle.c)
* ``Reference`` — oracle/_ref/libintzip_ref.so, the reference library compiled
                  from /root/reference/proj/core/src by oracle/Makefile

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libintzip_ref.so")

CHUNK_DTYPE = np.dtype([("word_off", "<u8"), ("n_words", "<u4"), ("n", "<u4"),
                        ("out_off", "<u8")])
CODECS = {"simdbp128": (0, 1), "simdbp128-s4": (0, 2), "simdfastpfor": (1, 1),
          "simdfastpfor-s4": (1, 2), "simdbp128-d2": (0, 3), "simdbp128-dm": (0, 4),
          "simdfastpfor-d2": (1, 3), "simdfastpfor-dm": (1, 4),
          "bp32": (2, 1), "bp32-s4": (2, 2), "fastpfor": (3, 1), "fastpfor-s4": (3, 2),
          "simplepfor": (4, 1), "simplepfor-s4": (4, 2)}


def build() -> None:
    """Compile the oracle (and the reference shim where the sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a):
    return a.ctypes.data


class Oracle:
    """The C restatement; statuses are izg_status codes."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        self.L = L = C.CDLL(ORACLE_SO)
        vp, sz = C.c_void_p, C.c_size_t
        L.orc_max_bitwidth.restype = C.c_uint32
        L.orc_max_bitwidth.argtypes = [vp, sz]
        L.orc_unpack_vertical128.argtypes = [vp, C.c_uint32, vp]
        L.orc_pack_vertical128.argtypes = [vp, C.c_uint32, vp]
        L.orc_delta_decode.argtypes = [C.c_int, vp, sz]
        L.orc_delta_encode.restype = C.c_int
        L.orc_delta_encode.argtypes = [C.c_int, vp, sz, C.c_int]
        L.orc_vbyte_encode.restype = sz
        L.orc_vbyte_encode.argtypes = [vp, sz, vp]
        L.orc_vbyte_decode.restype = C.c_int
        L.orc_vbyte_decode.argtypes = [vp, sz, vp, sz, C.POINTER(sz)]
        L.orc_histogram_of_widths.argtypes = [vp, sz, vp]
        L.orc_fastpfor_cost_bits.restype = C.c_uint64
        L.orc_fastpfor_cost_bits.argtypes = [vp, C.c_uint32, C.c_uint32]
        L.orc_fastpfor_choose_width.argtypes = [vp, C.c_uint32, C.POINTER(C.c_uint32),
                                                C.POINTER(C.c_uint32)]
        L.orc_encode_bound.restype = sz
        L.orc_encode_bound.argtypes = [C.c_int, sz]
        L.orc_encode_deltas.restype = sz
        L.orc_encode_deltas.argtypes = [C.c_int, vp, sz, vp]
        L.orc_decode_deltas.restype = C.c_int
        L.orc_decode_deltas.argtypes = [C.c_int, vp, sz, vp, sz, C.POINTER(sz)]
        L.orc_encode_chunk.restype = sz
        L.orc_encode_chunk.argtypes = [C.c_int, C.c_int, vp, C.c_uint32, vp, C.c_int]
        L.orc_decode_chunk.restype = C.c_int
        L.orc_decode_chunk.argtypes = [C.c_int, C.c_int, vp, sz, C.c_uint32, vp]

    def max_bitwidth(self, v):
        v = np.ascontiguousarray(v, dtype=np.uint32)
        return self.L.orc_max_bitwidth(_p(v), len(v))

    def unpack_vertical128(self, words, b):
        words = np.ascontiguousarray(words, dtype=np.uint32)
        out = np.zeros(128, dtype=np.uint32)
        self.L.orc_unpack_vertical128(_p(words), b, _p(out))
        return out

    def pack_vertical128(self, values, b):
        values = np.ascontiguousarray(values, dtype=np.uint32)
        out = np.zeros(max(4 * b, 1), dtype=np.uint32)
        self.L.orc_pack_vertical128(_p(values), b, _p(out))
        return out[:4 * b]

    def delta_decode(self, delta, v):
        v = np.array(v, dtype=np.uint32)
        self.L.orc_delta_decode(delta, _p(v), len(v))
        return v

    def delta_encode(self, delta, v, allow_wrap=False):
        v = np.array(v, dtype=np.uint32)
        if self.L.orc_delta_encode(delta, _p(v), len(v), int(allow_wrap)):
            raise ValueError("delta encode: input is not nondecreasing")
        return v

    def vbyte_encode(self, v):
        v = np.ascontiguousarray(v, dtype=np.uint32)
        out = np.zeros(5 * len(v) + 1, dtype=np.uint8)
        n = self.L.orc_vbyte_encode(_p(v), len(v), _p(out))
        return out[:n]

    def vbyte_decode(self, b, count):
        b = np.ascontiguousarray(b, dtype=np.uint8)
        out = np.zeros(max(count, 1), dtype=np.uint32)
        used = C.c_size_t()
        st = self.L.orc_vbyte_decode(_p(b), len(b), _p(out), count, C.byref(used))
        return st, out[:count], used.value

    def choose_width(self, hist33, block_len):
        h = np.ascontiguousarray(hist33, dtype=np.uint32)
        b, m = C.c_uint32(), C.c_uint32()
        self.L.orc_fastpfor_choose_width(_p(h), block_len, C.byref(b), C.byref(m))
        return b.value, m.value

    def cost_bits(self, hist33, block_len, b):
        h = np.ascontiguousarray(hist33, dtype=np.uint32)
        return self.L.orc_fastpfor_cost_bits(_p(h), block_len, b)

    def histogram(self, v):
        v = np.ascontiguousarray(v, dtype=np.uint32)
        h = np.zeros(33, dtype=np.uint32)
        self.L.orc_histogram_of_widths(_p(v), len(v), _p(h))
        return h

    def encode_deltas(self, name, deltas):
        codec = CODECS[name][0]
        deltas = np.ascontiguousarray(deltas, dtype=np.uint32)
        out = np.zeros(self.L.orc_encode_bound(codec, len(deltas)) + 64, dtype=np.uint32)
        n = self.L.orc_encode_deltas(codec, _p(deltas), len(deltas), _p(out))
        if n == C.c_size_t(-1).value:
            raise ValueError("count")
        return out[:n]

    def decode_deltas(self, name, words, count):
        codec = CODECS[name][0]
        words = np.ascontiguousarray(words, dtype=np.uint32)
        out = np.zeros(max(count, 1), dtype=np.uint32)
        used = C.c_size_t()
        st = self.L.orc_decode_deltas(codec, _p(words) if len(words) else None, len(words),
                                      _p(out), count, C.byref(used))
        return st, out[:count], used.value

    def encode_chunk(self, name, values, allow_wrap=False):
        codec, delta = CODECS[name]
        values = np.ascontiguousarray(values, dtype=np.uint32)
        out = np.zeros(self.L.orc_encode_bound(codec, len(values)) + 256, dtype=np.uint32)
        n = self.L.orc_encode_chunk(codec, delta, _p(values), len(values), _p(out),
                                    int(allow_wrap))
        if n == C.c_size_t(-1).value:
            raise ValueError("delta encode: input is not nondecreasing")
        return out[:n]

    def decode_chunk(self, name, payload, n):
        codec, delta = CODECS[name]
        payload = np.ascontiguousarray(payload, dtype=np.uint32)
        out = np.zeros(max(n, 1), dtype=np.uint32)
        st = self.L.orc_decode_chunk(codec, delta, _p(payload) if len(payload) else None,
                                     len(payload), n, _p(out))
        return st, out[:n]

    def encode_array(self, name, values, allow_wrap=False):
        values = np.ascontiguousarray(values, dtype=np.uint32)
        return [(min(65536, len(values) - o),
                 self.encode_chunk(name, values[o:o + 65536], allow_wrap))
                for o in range(0, len(values), 65536)]

    def decode_array(self, name, chunks):
        outs = []
        for n, payload in chunks:
            st, out = self.decode_chunk(name, payload, n)
            if st:
                return st, None
            outs.append(out)
        return 0, (np.concatenate(outs) if outs else np.zeros(0, np.uint32))


class RefError(Exception):
    def __init__(self, code, what):
        self.code, self.what = code, what
        super().__init__(f"[{code}] {what}")


class Reference:
    """The reference library itself (compiled from source); raises RefError
    with code 1 (CorruptError), 2 (invalid_argument) or 3 (other)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        self.L = L = C.CDLL(REF_SO)
        vp, u64, u32 = C.c_void_p, C.c_uint64, C.c_uint32
        cp = C.c_char_p
        L.izr_encode_array.restype = C.c_int
        L.izr_encode_array.argtypes = [cp, vp, u64, vp, u64, vp, u32, C.POINTER(u64),
                                       C.POINTER(u32), C.c_char_p, C.c_int]
        L.izr_encode_chunk_wrapping.restype = C.c_int
        L.izr_encode_chunk_wrapping.argtypes = [cp, vp, u32, vp, u64, C.POINTER(u64), C.c_char_p,
                                                C.c_int]
        L.izr_decode_array.restype = C.c_int
        L.izr_decode_array.argtypes = [cp, vp, vp, u32, vp, u64, C.c_char_p, C.c_int]
        L.izr_encode_deltas.restype = C.c_int
        L.izr_encode_deltas.argtypes = [cp, vp, u64, vp, u64, C.POINTER(u64), C.c_char_p, C.c_int]
        L.izr_decode_deltas.restype = C.c_int
        L.izr_decode_deltas.argtypes = [cp, vp, u64, vp, u64, C.POINTER(u64), C.c_char_p, C.c_int]
        L.izr_unpack_vertical128.restype = C.c_int
        L.izr_unpack_vertical128.argtypes = [vp, u32, vp]
        L.izr_pack_vertical128.restype = C.c_int
        L.izr_pack_vertical128.argtypes = [vp, u32, vp, C.c_int]
        L.izr_max_bitwidth.restype = u32
        L.izr_max_bitwidth.argtypes = [vp, u64]
        L.izr_delta.restype = C.c_int
        L.izr_delta.argtypes = [C.c_int, C.c_int, vp, u64]
        L.izr_vbyte_encode.restype = C.c_int
        L.izr_vbyte_encode.argtypes = [vp, u64, vp, C.POINTER(u64)]
        L.izr_vbyte_decode.restype = C.c_int
        L.izr_vbyte_decode.argtypes = [vp, u64, vp, u64, C.POINTER(u64), C.c_char_p, C.c_int]
        L.izr_choose_width.restype = C.c_int
        L.izr_choose_width.argtypes = [vp, u32, C.POINTER(u32), C.POINTER(u32), C.POINTER(u64)]
        L.izr_gen.restype = C.c_int
        L.izr_gen.argtypes = [C.c_int, u64, u64, u64, vp]
        L.izr_batch_create.restype = vp
        L.izr_batch_create.argtypes = [cp, vp, vp, u32]
        L.izr_batch_decode.restype = C.c_double
        L.izr_batch_decode.argtypes = [vp, u32, u32, C.c_int]
        L.izr_batch_output.restype = C.c_int
        L.izr_batch_output.argtypes = [vp, u32, vp]
        L.izr_batch_free.restype = None
        L.izr_batch_free.argtypes = [vp]
        L.izr_batch_new.restype = vp
        L.izr_batch_new.argtypes = [cp]
        L.izr_batch_adopt.restype = None
        L.izr_batch_adopt.argtypes = [vp, vp, C.c_int]
        L.izr_batch_size.restype = u32
        L.izr_batch_size.argtypes = [vp]
        L.izr_batch_payload_words.restype = u64
        L.izr_batch_payload_words.argtypes = [vp]
        L.izr_batch_checksum.restype = None
        L.izr_batch_checksum.argtypes = [vp, u32, u32, u64, vp]
        L.izr_encode_batch.restype = vp
        L.izr_encode_batch.argtypes = [cp, vp, vp, vp, u32, C.c_int, C.c_int, C.c_char_p,
                                       C.c_int]
        L.izr_encoded_size.restype = None
        L.izr_encoded_size.argtypes = [vp, C.c_int, C.POINTER(u64), C.POINTER(u32)]
        L.izr_encoded_copy.restype = None
        L.izr_encoded_copy.argtypes = [vp, C.c_int, vp, vp]
        L.izr_encoded_free.restype = None
        L.izr_encoded_free.argtypes = [vp]
        # the bench/test input generator (harness/csrc/datagen.cpp) compiled in
        L.izh_gen_arrays.restype = C.c_int
        L.izh_gen_arrays.argtypes = [C.c_int, u32, u32, u32, u32, u64, u32, C.c_int, vp, vp]
        L.izr_container_write_encoded.restype = C.c_int
        L.izr_container_write_encoded.argtypes = [cp, vp, vp, vp, u32, vp, u64, C.POINTER(u64),
                                                  C.c_char_p, C.c_int]
        L.izr_container_write_raw.restype = C.c_int
        L.izr_container_write_raw.argtypes = [vp, vp, vp, u32, vp, u64, C.POINTER(u64),
                                              C.c_char_p, C.c_int]
        L.izr_container_read_encoded.restype = C.c_int
        L.izr_container_read_encoded.argtypes = [vp, u64, C.c_char_p, C.c_int, vp, u64, vp, u32,
                                                 vp, u32, C.POINTER(u32), C.POINTER(u32),
                                                 C.c_char_p, C.c_int]
        L.izr_container_read_raw.restype = C.c_int
        L.izr_container_read_raw.argtypes = [vp, u64, vp, u64, vp, u32, C.POINTER(u32),
                                             C.c_char_p, C.c_int]

    @staticmethod
    def _check(rc, err):
        if rc:
            raise RefError(rc, err.value.decode())

    # ---- container.cpp -------------------------------------------------------

    @staticmethod
    def _arrays(arrays):
        lens = np.array([len(a) for a in arrays], dtype=np.uint32)
        offs = np.zeros(len(arrays), dtype=np.uint64)
        if len(arrays) > 1:
            offs[1:] = np.cumsum(lens[:-1], dtype=np.uint64)
        flat = (np.concatenate([np.asarray(a, np.uint32) for a in arrays])
                if arrays and lens.sum() else np.zeros(1, np.uint32))
        return flat, offs, lens

    def _write(self, fn, *args):
        n = C.c_uint64()
        err = C.create_string_buffer(256)
        self._check(fn(*args, None, 0, C.byref(n), err, 256), err)
        buf = np.zeros(max(n.value, 1), dtype=np.uint8)
        self._check(fn(*args, _p(buf), len(buf), C.byref(n), err, 256), err)
        return buf[:n.value].tobytes()

    def container_write_encoded(self, name, arrays):
        flat, offs, lens = self._arrays(arrays)
        return self._write(self.L.izr_container_write_encoded, name.encode(), _p(flat), _p(offs),
                           _p(lens) if len(lens) else None, len(arrays))

    def container_write_raw(self, arrays):
        flat, offs, lens = self._arrays(arrays)
        return self._write(self.L.izr_container_write_raw, _p(flat), _p(offs),
                           _p(lens) if len(lens) else None, len(arrays))

    def container_read_encoded(self, data):
        """(codec name, [[(original_length, payload words), ...] per array])."""
        buf = np.frombuffer(bytes(data) + b"\0", dtype=np.uint8)
        cap_w = len(data) // 4 + 1
        words = np.zeros(cap_w, dtype=np.uint32)
        table = np.zeros(cap_w, dtype=CHUNK_DTYPE)
        c0 = np.zeros(len(data) // 8 + 2, dtype=np.uint32)
        name = C.create_string_buffer(300)
        na, nc = C.c_uint32(), C.c_uint32()
        err = C.create_string_buffer(256)
        rc = self.L.izr_container_read_encoded(_p(buf), len(data), name, 300, _p(words), cap_w,
                                               _p(table), len(table), _p(c0), len(c0),
                                               C.byref(na), C.byref(nc), err, 256)
        self._check(rc, err)
        out = []
        for a in range(na.value):
            out.append([(int(t["n"]), words[int(t["word_off"]):int(t["word_off"]) +
                                            int(t["n_words"])].copy())
                        for t in table[c0[a]:c0[a + 1]]])
        return name.value.decode(), out

    def container_read_raw(self, data):
        buf = np.frombuffer(bytes(data) + b"\0", dtype=np.uint8)
        cap = len(data) // 4 + 1
        vals = np.zeros(cap, dtype=np.uint32)
        lens = np.zeros(len(data) // 8 + 1, dtype=np.uint32)
        na = C.c_uint32()
        err = C.create_string_buffer(256)
        rc = self.L.izr_container_read_raw(_p(buf), len(data), _p(vals), cap, _p(lens), len(lens),
                                           C.byref(na), err, 256)
        self._check(rc, err)
        out, pos = [], 0
        for n in lens[:na.value]:
            out.append(vals[pos:pos + int(n)].copy())
            pos += int(n)
        return out

    def encode_array(self, name, values):
        values = np.ascontiguousarray(values, dtype=np.uint32)
        nchunks = (len(values) + 65535) // 65536
        cap = 2 * len(values) + 1024 * (nchunks + 1)
        words = np.zeros(cap, dtype=np.uint32)
        table = np.zeros(max(nchunks, 1), dtype=CHUNK_DTYPE)
        nw, nc = C.c_uint64(), C.c_uint32()
        err = C.create_string_buffer(256)
        rc = self.L.izr_encode_array(name.encode(), _p(values), len(values), _p(words), cap,
                                     _p(table), len(table), C.byref(nw), C.byref(nc), err, 256)
        self._check(rc, err)
        table = table[:nc.value]
        return [(int(t["n"]), words[int(t["word_off"]):int(t["word_off"]) + int(t["n_words"])].copy())
                for t in table]

    def encode_chunk_wrapping(self, name, values):
        values = np.ascontiguousarray(values, dtype=np.uint32)
        cap = 2 * len(values) + 1024
        words = np.zeros(cap, dtype=np.uint32)
        nw = C.c_uint64()
        err = C.create_string_buffer(256)
        rc = self.L.izr_encode_chunk_wrapping(name.encode(), _p(values), len(values), _p(words),
                                              cap, C.byref(nw), err, 256)
        self._check(rc, err)
        return words[:nw.value].copy()

    def decode_array(self, name, chunks):
        """chunks: list of (n, payload); raises RefError like decode_array."""
        payloads = [np.ascontiguousarray(p, dtype=np.uint32) for _, p in chunks]
        words = np.concatenate(payloads) if payloads else np.zeros(1, np.uint32)
        if len(words) == 0:
            words = np.zeros(1, np.uint32)
        table = np.zeros(max(len(chunks), 1), dtype=CHUNK_DTYPE)
        off = 0
        for i, (n, p) in enumerate(chunks):
            table[i] = (off, len(p), n, 0)
            off += len(p)
        total = sum(n for n, _ in chunks)
        out = np.zeros(max(total, 1), dtype=np.uint32)
        err = C.create_string_buffer(256)
        rc = self.L.izr_decode_array(name.encode(), _p(words), _p(table), len(chunks), _p(out),
                                     len(out), err, 256)
        self._check(rc, err)
        return out[:total]

    def encode_deltas(self, name, deltas):
        deltas = np.ascontiguousarray(deltas, dtype=np.uint32)
        cap = 2 * len(deltas) + 1024
        words = np.zeros(cap, dtype=np.uint32)
        nw = C.c_uint64()
        err = C.create_string_buffer(256)
        rc = self.L.izr_encode_deltas(name.encode(), _p(deltas), len(deltas), _p(words), cap,
                                      C.byref(nw), err, 256)
        self._check(rc, err)
        return words[:nw.value].copy()

    def decode_deltas(self, name, words, count):
        words = np.ascontiguousarray(words, dtype=np.uint32)
        buf = words if len(words) else np.zeros(1, np.uint32)
        out = np.zeros(max(count, 1), dtype=np.uint32)
        used = C.c_uint64()
        err = C.create_string_buffer(256)
        rc = self.L.izr_decode_deltas(name.encode(), _p(buf), len(words), _p(out), count,
                                      C.byref(used), err, 256)
        self._check(rc, err)
        return out[:count], used.value

    def unpack_vertical128(self, words, b):
        words = np.ascontiguousarray(words, dtype=np.uint32)
        buf = words if len(words) else np.zeros(4, np.uint32)
        out = np.zeros(128, dtype=np.uint32)
        if self.L.izr_unpack_vertical128(_p(buf), b, _p(out)):
            raise RefError(2, "width")
        return out

    def pack_vertical128(self, values, b, masked=False):
        values = np.ascontiguousarray(values, dtype=np.uint32)
        out = np.zeros(4 * 33, dtype=np.uint32)
        rc = self.L.izr_pack_vertical128(_p(values), b, _p(out), int(masked))
        if rc:
            raise RefError(rc, "pack")
        return out[:4 * b]

    def max_bitwidth(self, v):
        v = np.ascontiguousarray(v, dtype=np.uint32)
        return self.L.izr_max_bitwidth(_p(v) if len(v) else None, len(v))

    def delta(self, encode, stride4, v):
        v = np.array(v, dtype=np.uint32)
        buf = v if len(v) else np.zeros(1, np.uint32)
        rc = self.L.izr_delta(int(encode), int(stride4), _p(buf), len(v))
        if rc:
            raise RefError(rc, "delta")
        return buf[:len(v)]

    def vbyte_encode(self, v):
        v = np.ascontiguousarray(v, dtype=np.uint32)
        out = np.zeros(5 * len(v) + 1, dtype=np.uint8)
        n = C.c_uint64()
        self.L.izr_vbyte_encode(_p(v) if len(v) else None, len(v), _p(out), C.byref(n))
        return out[:n.value]

    def vbyte_decode(self, b, count):
        b = np.ascontiguousarray(b, dtype=np.uint8)
        buf = b if len(b) else np.zeros(1, np.uint8)
        out = np.zeros(max(count, 1), dtype=np.uint32)
        used = C.c_uint64()
        err = C.create_string_buffer(256)
        rc = self.L.izr_vbyte_decode(_p(buf), len(b), _p(out), count, C.byref(used), err, 256)
        self._check(rc, err)
        return out[:count], used.value

    def choose_width(self, hist33, block_len):
        h = np.ascontiguousarray(hist33, dtype=np.uint32)
        b, m, c = C.c_uint32(), C.c_uint32(), C.c_uint64()
        self.L.izr_choose_width(_p(h), block_len, C.byref(b), C.byref(m), C.byref(c))
        return b.value, m.value, c.value

    def gen(self, model, n, rng, seed):
        out = np.zeros(max(n, 1), dtype=np.uint32)
        if self.L.izr_gen({"uniform": 0, "cluster": 1}[model], n, rng, seed, _p(out)):
            raise RefError(2, "gen")
        return out[:n]

    # ---- harness generator compiled into the shim (reference arm inputs) ----
    def gen_arrays(self, model, count, n, d, seed, *, rate_ppm=0, threads=1, out=None):
        """Same arrays as harness.gen_arrays (the same source, datagen.cpp)."""
        d_lo, d_hi = (d, d) if np.isscalar(d) else d
        if out is None:
            out = np.empty((count, n), dtype=np.uint32)
        dd = np.empty(count, dtype=np.uint32)
        models = {"uniform": 0, "cluster": 1, "geometric": 2, "raw": 3}
        if self.L.izh_gen_arrays(models[model], count, n, d_lo, d_hi, seed, rate_ppm, threads,
                                 _p(out), _p(dd)):
            raise RefError(2, "gen_arrays: bad arguments")
        return out, dd

    # ---- threaded batch encode with the reference encoder ----
    def _encode_handle(self, name, values, value_off, counts, wrap, threads):
        values = np.ascontiguousarray(values, dtype=np.uint32)
        value_off = np.ascontiguousarray(value_off, dtype=np.uint64)
        counts = np.ascontiguousarray(counts, dtype=np.uint32)
        err = C.create_string_buffer(256)
        h = self.L.izr_encode_batch(name.encode(), _p(values), _p(value_off), _p(counts),
                                    len(counts), int(wrap), threads, err, 256)
        if not h:
            raise RefError(2, err.value.decode())
        return h

    def encode_batch(self, name, values, value_off, counts, *, wrap=False, threads=1, phase=None):
        """Arrays values[value_off[i]:+counts[i]] through encode_array (or the
        wrapping rule, wrap=True), on `threads` threads.  Returns (words,
        table): chunk payloads placed with word 0 at `phase` mod 4 (default:
        izg_layout_chunks' placement for the codec), outputs back to back."""
        if phase is None:
            phase = 3 if name.startswith("simdfastpfor") else 0
        h = self._encode_handle(name, values, value_off, counts, wrap, threads)
        try:
            nw, nc = C.c_uint64(), C.c_uint32()
            self.L.izr_encoded_size(h, phase, C.byref(nw), C.byref(nc))
            words = np.empty(nw.value, dtype=np.uint32)
            table = np.empty(nc.value, dtype=CHUNK_DTYPE)
            self.L.izr_encoded_copy(h, phase, _p(words), _p(table))
        finally:
            self.L.izr_encoded_free(h)
        return words, table

    def batch_new(self, name):
        return RefBatch(self, self.L.izr_batch_new(name.encode()), 0)

    # ---- timed batch decode (reference arm / cpu_baseline) ----
    def batch(self, name, words, table):
        words = np.ascontiguousarray(words, dtype=np.uint32)
        table = np.ascontiguousarray(table, dtype=CHUNK_DTYPE)
        return RefBatch(self, self.L.izr_batch_create(name.encode(), _p(words), _p(table),
                                                      len(table)), len(table))


class RefBatch:
    def __init__(self, ref, handle, n):
        self.ref, self.h, self.n = ref, handle, n

    def add(self, name, values, value_off, counts, *, wrap=False, threads=1):
        """Encode arrays with the reference (threaded) and append them."""
        h = self.ref._encode_handle(name, values, value_off, counts, wrap, threads)
        self.ref.L.izr_batch_adopt(self.h, h, threads)
        self.n = self.ref.L.izr_batch_size(self.h)

    def payload_words(self) -> int:
        return int(self.ref.L.izr_batch_payload_words(self.h))

    def checksum(self, first=0, count=None, base=0):
        count = self.n - first if count is None else count
        out = np.zeros(2, dtype=np.uint64)
        self.ref.L.izr_batch_checksum(self.h, first, count, base, _p(out))
        return int(out[0]), int(out[1])

    def decode(self, first=0, count=None, threads=1) -> float:
        count = self.n - first if count is None else count
        t = self.ref.L.izr_batch_decode(self.h, first, count, threads)
        if t < 0:
            raise RefError(1, "decode failed in batch")
        return t

    def output(self, i, n):
        out = np.zeros(n, dtype=np.uint32)
        self.ref.L.izr_batch_output(self.h, i, _p(out))
        return out

    def close(self):
        if self.h:
            self.ref.L.izr_batch_free(self.h)
            self.h = None

    def __del__(self):
        self.close()
