"""Device-resident batches for izg_decode (stream-ordered, no host sync).

torch provides device memory and streams only (plumbing); the decode itself is
the fused kernel behind the C ABI.
"""
from __future__ import annotations

import numpy as np

from . import _native as N
from .codec import Codec, Encoded, raise_for_status


class DeviceBatch:
    """An Encoded batch resident in HBM plus its output and status buffers.

    indexed=True gives SIMD-FastPFOR batches a decode workspace, so decode()
    runs izg_decode_ws's two-launch path (page index pass + table-driven
    decode); indexed=False keeps the single fused launch of izg_decode.
    materialize=False allocates no output (for decode_intersect_device).
    relay_long_only=False keeps the SIMD-BP128 relay workspace for batches of short
    chunks too (tests).
    split=False sizes the workspace for the page index only, so small batches
    keep one warp per chunk instead of the split kernel (csrc/split.cuh)."""

    def __init__(self, codec: Codec, enc: Encoded, device=None, *, raw: bool = False,
                 out=None, indexed: bool = True, materialize: bool = True,
                 split: bool = True, relay_long_only: bool = True):
        import torch

        self.torch = torch
        self.codec = codec
        self.delta = N.DELTA_NONE if raw else codec.delta
        self.device = torch.device(device or "cuda")
        self.n_chunks = len(enc.table)
        self.n_out = enc.n_out
        self.payload_words = enc.payload_words
        self.words = torch.from_numpy(enc.words.view(np.int32)).to(self.device)
        self.table = torch.from_numpy(enc.table.view(np.uint8)).to(self.device)
        if not materialize:  # decode_intersect_device only: no output buffer
            self.out = torch.empty(1, dtype=torch.int32, device=self.device)
        elif out is not None:
            assert out.numel() >= self.n_out and out.dtype == torch.int32
            self.out = out
        else:
            self.out = torch.empty(max(self.n_out, 1), dtype=torch.int32, device=self.device)
        self.status = torch.full((max(self.n_chunks, 1),), -1, dtype=torch.int32,
                                 device=self.device)
        self.consumed = torch.zeros(max(self.n_chunks, 1), dtype=torch.int32,
                                    device=self.device)
        self.sums = torch.zeros(2, dtype=torch.int64, device=self.device)
        L = N.lib()
        ws = 0
        if indexed:
            ws = (L.izg_decode_workspace_size(codec.codec, self.n_chunks) if split
                  else L.izg_decode_index_workspace_size(codec.codec, self.n_chunks))
            # SIMD-BP128 batches of 2,432+ chunks: the workspace selects the relay kernel,
            # which pays for long chunks only (4-12 % at 65,536 integers per chunk, 5-15 %
            # lost on chunks of a few thousand: tools/relay_short.py)
            if (relay_long_only and codec.codec == N.SIMDBP128 and self.n_chunks >= 2432
                    and self.n_out < 32768 * self.n_chunks):
                ws = 0
        self.workspace = (torch.empty(ws, dtype=torch.uint8, device=self.device)
                          if ws else None)

    @property
    def launches_per_decode(self) -> int:
        """Kernels one decode() launches (memsets excluded): the indexed
        SIMD-FastPFOR path runs the page index pass, then the decode."""
        return 2 if self.workspace is not None else 1

    @property
    def algorithmic_bytes(self) -> int:
        """Compressed bytes read + 4 B per decoded integer."""
        return 4 * self.payload_words + 4 * self.n_out

    def decode(self, stream=None) -> None:
        s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        if self.workspace is not None:
            rc = N.lib().izg_decode_ws(self.codec.codec, self.delta, N.ptr(self.words),
                                       N.ptr(self.table), self.n_chunks, N.ptr(self.out),
                                       N.ptr(self.status), N.ptr(self.consumed),
                                       N.ptr(self.workspace), self.workspace.numel(),
                                       s.cuda_stream)
        else:
            rc = N.lib().izg_decode(self.codec.codec, self.delta, N.ptr(self.words),
                                    N.ptr(self.table), self.n_chunks, N.ptr(self.out),
                                    N.ptr(self.status), N.ptr(self.consumed), s.cuda_stream)
        if rc != N.SUCCESS:
            raise RuntimeError(f"izg_decode failed: {rc}")

    def decode_phase(self, phase: int, stream=None) -> None:
        """izg_decode_ws_phase: 1 = the page index pass alone, 2 = the decode
        alone (after phase 1 on the same batch, stream-ordered), 0 = both."""
        s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        ws = self.workspace
        rc = N.lib().izg_decode_ws_phase(self.codec.codec, self.delta, N.ptr(self.words),
                                         N.ptr(self.table), self.n_chunks, N.ptr(self.out),
                                         N.ptr(self.status), N.ptr(self.consumed),
                                         N.ptr(ws) if ws is not None else None,
                                         ws.numel() if ws is not None else 0, phase,
                                         s.cuda_stream)
        if rc != N.SUCCESS:
            raise RuntimeError(f"izg_decode_ws_phase failed: {rc}")

    def checksum(self, stream=None) -> tuple[int, int]:
        s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        rc = N.lib().izg_checksum(N.ptr(self.out), self.n_out, N.ptr(self.sums), s.cuda_stream)
        if rc != N.SUCCESS:
            raise RuntimeError(f"izg_checksum failed: {rc}")
        v = self.sums.cpu().numpy().view(np.uint64)
        return int(v[0]), int(v[1])

    def statuses(self) -> np.ndarray:
        return self.status[:self.n_chunks].cpu().numpy()

    def check(self) -> None:
        st = self.statuses()
        bad = np.nonzero(st)[0]
        if len(bad):
            raise_for_status(int(st[bad[0]]), int(bad[0]))

    def output(self) -> np.ndarray:
        return self.out[:self.n_out].cpu().numpy().view(np.uint32)


def host_checksum(values: np.ndarray, base_index: int = 0) -> tuple[int, int]:
    """izg_checksum on the host: sum (w+1)(2i+1) mod 2^64, xor of words."""
    v = np.ascontiguousarray(values, dtype=np.uint32).reshape(-1).astype(np.uint64)
    i = np.arange(base_index, base_index + len(v), dtype=np.uint64)
    with np.errstate(over="ignore"):
        s = int(np.sum((v + np.uint64(1)) * (np.uint64(2) * i + np.uint64(1)), dtype=np.uint64))
    x = int(np.bitwise_xor.reduce(v)) if len(v) else 0
    return s, x


def encode_on_device(codec: Codec, values, value_off, counts, *, allow_wrap: bool = False,
                     raw: bool = False, device=None):
    """GPU encoder (izg_encode): returns (Encoded with host copies, statuses).

    Chunks are placed in slots of izg_encode_bound words (4-word aligned), so
    the result satisfies izg_decode's placement contract as is."""
    import torch

    dev = torch.device(device or "cuda")
    L = N.lib()
    counts = np.ascontiguousarray(counts, dtype=np.uint32)
    value_off = np.ascontiguousarray(value_off, dtype=np.uint64)
    bounds = np.array([L.izg_encode_bound(codec.codec, int(n)) for n in counts], np.uint64)
    slots = (bounds + 3) // 4 * 4
    word_off = np.concatenate([[0], np.cumsum(slots)[:-1]]).astype(np.uint64) if len(slots) else slots
    total = int(slots.sum()) + 4
    table = np.zeros(len(counts), dtype=N.CHUNK_DTYPE)
    table["word_off"] = word_off
    table["n"] = counts
    table["out_off"] = value_off
    vals = values if isinstance(values, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(values, dtype=np.uint32).view(np.int32))
    vals = vals.to(dev)
    d_table = torch.from_numpy(table.view(np.uint8)).to(dev)
    d_words = torch.zeros(total, dtype=torch.int32, device=dev)
    d_status = torch.full((max(len(counts), 1),), -1, dtype=torch.int32, device=dev)
    delta = N.DELTA_NONE if raw else codec.delta
    s = torch.cuda.current_stream(dev)
    rc = L.izg_encode(codec.codec, delta, N.ptr(vals), N.ptr(d_table), len(counts),
                      N.ptr(d_words), N.ptr(d_status), int(allow_wrap), s.cuda_stream)
    if rc != N.SUCCESS:
        raise RuntimeError(f"izg_encode failed: {rc}")
    out_table = d_table.cpu().numpy().view(N.CHUNK_DTYPE).copy()
    # as a decode batch the outputs go back to back
    out_table["out_off"] = value_off
    enc = Encoded(d_words.cpu().numpy().view(np.uint32), out_table)
    return enc, d_status[:len(counts)].cpu().numpy()


def intersect_device(a, b, stream=None):
    """Sorted intersection (numpy.intersect1d semantics) of two nondecreasing
    int32/uint32 CUDA tensors on the device (izg_intersect_sorted); returns a
    CUDA tensor of the common values.  The consumer of SURVEY.md §8 f4."""
    import torch

    dev = a.device
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    na, nb = a.numel(), b.numel()
    out = torch.empty(max(min(na, nb), 1), dtype=torch.int32, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(N.lib().izg_intersect_workspace_size(na, nb), dtype=torch.uint8, device=dev)
    rc = N.lib().izg_intersect_sorted(N.ptr(a) if na else None, na, N.ptr(b) if nb else None, nb,
                                      N.ptr(out), N.ptr(count), N.ptr(ws), ws.numel(),
                                      s.cuda_stream)
    if rc != N.SUCCESS:
        raise RuntimeError(f"izg_intersect_sorted failed: {rc}")
    return out[:int(count.item())]


def decode_intersect_device(batch: "DeviceBatch", s_list, stream=None):
    """Fused decode -> intersect (izg_decode_intersect): decodes `batch`'s
    chunks and intersects them with the nondecreasing CUDA tensor `s_list`
    without writing the decoded integers anywhere (each tile is merged
    against s_list in shared memory).  Returns a CUDA tensor of the distinct
    common values, ascending; per-chunk statuses land in batch.status."""
    import torch

    dev = s_list.device
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    L = N.lib()
    ns = s_list.numel()
    out = torch.empty(max(ns, 1), dtype=torch.int32, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(L.izg_decode_intersect_workspace_size(ns), dtype=torch.uint8, device=dev)
    rc = L.izg_decode_intersect(batch.codec.codec, batch.delta, N.ptr(batch.words),
                                N.ptr(batch.table), batch.n_chunks,
                                N.ptr(s_list) if ns else None, ns, N.ptr(out), N.ptr(count),
                                N.ptr(batch.status), N.ptr(ws), ws.numel(), s.cuda_stream)
    if rc != N.SUCCESS:
        raise RuntimeError(f"izg_decode_intersect failed: {rc}")
    return out[:int(count.item())]


def intersect(codec: Codec, enc_a: Encoded, enc_b: Encoded, device=None,
              fused: bool = True) -> np.ndarray:
    """Decode two encoded arrays (posting lists) on the GPU and intersect them
    there; only the intersection is copied back (numpy.intersect1d result).

    fused=True (default): the shorter list is decoded to HBM and the longer
    one goes through izg_decode_intersect, so it is never materialised.
    fused=False: both are decoded, then izg_intersect_sorted."""
    if fused:
        short, long_ = (enc_a, enc_b) if enc_a.n_out <= enc_b.n_out else (enc_b, enc_a)
        bs = DeviceBatch(codec, short, device)
        bl = DeviceBatch(codec, long_, device, materialize=False, indexed=False)
        bs.decode()
        bs.check()
        r = decode_intersect_device(bl, bs.out[:bs.n_out])
        bl.check()
        return r.cpu().numpy().view(np.uint32)
    ba = DeviceBatch(codec, enc_a, device)
    bb = DeviceBatch(codec, enc_b, device)
    ba.decode()
    bb.decode()
    ba.check()
    bb.check()
    r = intersect_device(ba.out[:ba.n_out], bb.out[:bb.n_out])
    return r.cpu().numpy().view(np.uint32)
