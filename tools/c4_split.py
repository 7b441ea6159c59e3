"""Developer: C4 (2,048 pages, 10 % / 1 % outliers) — the page index pass and the
team decode timed separately (izg_decode_ws_phase 1 / 2) and together."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P
count = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
for rate in (100000, 10000):
    vals, _ = H.gen_arrays("geometric", count, 65536, 32, seed=1, rate_ppm=rate)
    codec = P.make_codec("simdfastpfor-s4")
    enc = H.encode_chunks(codec, vals.reshape(-1), np.arange(count, dtype=np.uint64) * 65536,
                          np.full(count, 65536, np.uint32), allow_wrap=True)
    b = P.DeviceBatch(codec, enc, split=False)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    for what, fn in (("index", lambda: b.decode_phase(1)), ("decode", lambda: b.decode_phase(2)),
                     ("both", lambda: b.decode())):
        t = []
        for _ in range(12):
            if what != "decode":
                flush.zero_()
            else:
                flush.zero_(); b.decode_phase(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            t.append(e0.elapsed_time(e1))
        res[what] = round(float(np.median(t[2:])), 4)
    b.check()
    print("rate_ppm", rate, "pages", count, res, flush=True)
