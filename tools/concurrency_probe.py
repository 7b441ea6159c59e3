"""Developer probe: does running the C5 step's two codecs concurrently beat
running them back to back?  SIMD-BP128 is HBM-bound and SIMD-FastPFOR
issue-bound (profiles/README.md), so co-resident CTAs of the two could
overlap.  Variants (each verified by checksum):

  serial   one stream, BP128 then FastPFOR (bench.py's step)
  two      BP128 on stream 1, FastPFOR on stream 2, separate outputs
  prioN    as `two`, BP128's stream at high priority
  sliceS   each codec's page table cut into S slices, slices alternate
           on the two streams (tails of one filled by the other)

usage: python tools/concurrency_probe.py [arrays]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1209_2137_b200 as P  # noqa: E402
from paper_1209_2137_b200 import _native as N  # noqa: E402


def main():
    n_arrays = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    wl = list(bench.WORKLOADS["c5"])
    wl[0] = n_arrays
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    t0 = time.time()
    encs, expect, _ = bench.build_inputs(P, tuple(wl), 0, n_arrays, os.cpu_count() or 1)
    print(f"prep {time.time() - t0:.1f}s", flush=True)
    L = N.lib()
    batches = {c: P.DeviceBatch(P.make_codec(c), encs[c], dev) for c in bench.CODECS}
    main_s = torch.cuda.current_stream(dev)
    s1 = torch.cuda.Stream(dev)
    s2 = torch.cuda.Stream(dev)
    lo_p, hi_p = torch.cuda.Stream.priority_range()
    s1h = torch.cuda.Stream(dev, priority=hi_p)

    def sliced(b, k, S, stream):
        n = b.n_chunks
        a0, a1 = n * k // S, n * (k + 1) // S
        row = b.table.numel() // n
        ws = b.workspace
        wsz = 0
        wp = 0
        if ws is not None:
            wsz = L.izg_decode_workspace_size(b.codec.codec, a1 - a0)
            wp = N.ptr(ws)  # slices on one stream run in order: one workspace each stream
        if ws is None:
            rc = L.izg_decode(b.codec.codec, b.delta, N.ptr(b.words), N.ptr(b.table) + row * a0,
                              a1 - a0, N.ptr(b.out), N.ptr(b.status) + 4 * a0,
                              N.ptr(b.consumed) + 4 * a0, stream.cuda_stream)
            assert rc == 0, rc
            return
        rc = L.izg_decode_ws(b.codec.codec, b.delta, N.ptr(b.words), N.ptr(b.table) + row * a0,
                             a1 - a0, N.ptr(b.out), N.ptr(b.status) + 4 * a0,
                             N.ptr(b.consumed) + 4 * a0, wp, wsz, stream.cuda_stream)
        assert rc == 0, rc

    bp, fp = batches["simdbp128-s4"], batches["simdfastpfor-s4"]

    def run(variant):
        if variant == "serial":
            bp.decode(main_s)
            fp.decode(main_s)
            return
        if variant.startswith("slice"):
            S = int(variant[5:])
            for st in (s1, s2):
                st.wait_stream(main_s)
            for k in range(S):
                sliced(bp, k, S, s1)
                sliced(fp, k, S, s2)
            main_s.wait_stream(s1)
            main_s.wait_stream(s2)
            return
        a = s1h if variant == "prio" else s1
        for st in (a, s2):
            st.wait_stream(main_s)
        if variant == "two_fpfirst":
            fp.decode(s2)
            bp.decode(a)
        else:
            bp.decode(a)
            fp.decode(s2)
        main_s.wait_stream(a)
        main_s.wait_stream(s2)

    ints = 2 * n_arrays * bench.N_INTS
    for v in ("serial", "two", "two_fpfirst", "prio", "slice2", "slice4", "slice8", "serial"):
        for _ in range(3):
            run(v)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 10
        e0.record(main_s)
        for _ in range(K):
            run(v)
        e1.record(main_s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        ok = all(b.checksum() == expect for b in (bp, fp))
        for b in (bp, fp):
            b.check()
        print(f"{v:12s} {ms:8.3f} ms/step  {ints / ms / 1e6:8.1f} G int/s  verified={ok}",
              flush=True)


if __name__ == "__main__":
    main()
