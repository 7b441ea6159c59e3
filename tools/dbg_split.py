import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1209_2137_b200 as P
for name, model, d, rate, count in [("simdbp128-s4", "cluster", 29, 0, 2048), ("simdfastpfor-s4", "geometric", 32, 100000, 1024)]:
    codec = P.make_codec(name)
    vals, _ = P.gen_arrays(model, count, 65536, d, seed=1, rate_ppm=rate)
    flat = vals.reshape(-1)
    enc = P.encode_chunks(codec, flat, np.arange(count, dtype=np.uint64) * 65536,
                          np.full(count, 65536, np.uint32), allow_wrap=model == "geometric")
    ws = P.DeviceBatch(codec, enc)
    for rep in range(4):
        ws.out.fill_(0)
        ws.decode(); torch.cuda.synchronize()
        ws.check()
        got = ws.output().reshape(count, 65536)
        bad = np.nonzero((got != vals).any(axis=1))[0]
        print(name, "rep", rep, "bad chunks", len(bad), bad[:10])
        for c in bad[:3]:
            diff = np.nonzero(got[c] != vals[c])[0]
            segs = np.unique(diff // 4096)
            print("  chunk", c, "n diff", len(diff), "segments", segs[:20], "first", diff[:4],
                  "delta", (got[c][diff[:8]].astype(np.int64) - vals[c][diff[:8]].astype(np.int64)))
