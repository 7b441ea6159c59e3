"""Developer: the SIMD-FastPFOR page index pass alone (izg_decode_ws_phase 1), C5 pages."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P
count = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
vals, _ = H.gen_arrays("cluster", count, 65536, (20, 29), seed=1)
codec = P.make_codec("simdfastpfor-s4")
enc = H.encode_chunks(codec, vals.reshape(-1), np.arange(count, dtype=np.uint64) * 65536, np.full(count, 65536, np.uint32))
b = P.DeviceBatch(codec, enc, split=False)
t = []
for _ in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.decode_phase(1); e1.record(); torch.cuda.synchronize()
    t.append(e0.elapsed_time(e1))
print(os.path.basename(os.environ.get("IZG_LIB_PATH", "default")), count, round(float(np.median(t)), 4))
