"""Time izg_decode_host (host buffers in/out) on a C5-like batch."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P
count = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
vals, _ = H.gen_arrays("cluster", count, 65536, (20, 29), seed=1)
flat = vals.reshape(-1)
offs = np.arange(count, dtype=np.uint64) * 65536
for name in ("simdbp128-s4", "simdfastpfor-s4"):
    codec = P.make_codec(name)
    e = H.encode_chunks(codec, flat, offs, np.full(count, 65536, np.uint32))
    hw = torch.empty(len(e.words), dtype=torch.int32, pin_memory=True)
    hw.numpy().view(np.uint32)[:] = e.words
    ho = torch.empty(e.n_out, dtype=torch.int32, pin_memory=True)
    st = np.zeros(len(e.table), np.int32)
    L = P._native.lib()
    def run():
        rc = L.izg_decode_host(codec.codec, codec.delta, hw.data_ptr(), len(e.words), P._native.ptr(e.table),
                               len(e.table), ho.data_ptr(), e.n_out, P._native.ptr(st))
        assert rc == 0, rc
    run()
    ts = []
    for _ in range(3):
        t = time.perf_counter(); run(); ts.append(time.perf_counter() - t)
    t = min(ts)
    assert np.array_equal(ho.numpy().view(np.uint32)[:65536], vals[0])
    print(name, "G ints/s", round(flat.size / t / 1e9, 2), "d2h GB/s", round(4 * flat.size / t / 1e9, 1),
          "h2d GB/s", round(4 * len(e.words) / t / 1e9, 1), "ms", round(t * 1e3, 1), flush=True)
