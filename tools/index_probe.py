"""Developer: SIMD-FastPFOR page index pass (izg_decode_ws_phase 1) and decode
(phase 2) timed separately, C5 data, by batch size."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P

counts = [int(x) for x in (sys.argv[1:] or ["2048", "8192", "32768"])]
vals, _ = H.gen_arrays("cluster", max(counts), 65536, (20, 29), seed=1)
flat = vals.reshape(-1)
codec = P.make_codec("simdfastpfor-s4")
for count in counts:
    enc = H.encode_chunks(codec, flat[:count * 65536], np.arange(count, dtype=np.uint64) * 65536,
                          np.full(count, 65536, np.uint32))
    b = P.DeviceBatch(codec, enc, split=False)
    for _ in range(3):
        b.decode()
    torch.cuda.synchronize(); b.check()
    t = {1: [], 2: []}
    for _ in range(10):
        for ph in (1, 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); b.decode_phase(ph); e1.record(); torch.cuda.synchronize()
            t[ph].append(e0.elapsed_time(e1))
    b.check()
    print(json.dumps({"lib": os.path.basename(os.environ.get("IZG_LIB_PATH", "default")), "pages": count,
                      "index_ms": round(float(np.median(t[1])), 4), "decode_ms": round(float(np.median(t[2])), 4)}), flush=True)
