"""Launch the decode kernel a few times on one config (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P

CFG = {
    "c1": ("simdbp128-s4", "cluster", 1024, 29, 0, False),
    "c1big": ("simdbp128-s4", "cluster", 8192, 29, 0, False),
    "raw0": ("simdbp128", "raw", 4096, 0, 0, True),
    "raw16": ("simdbp128", "raw", 4096, 16, 0, True),
    "c3": ("simdbp128-s4", "uniform", 4096, 26, 0, False),
    "c4": ("simdfastpfor-s4", "geometric", 2048, 32, 100000, False),
    "c5fp": ("simdfastpfor-s4", "cluster", 8192, (20, 29), 0, False),
    "c5bp": ("simdbp128-s4", "cluster", 8192, (20, 29), 0, False),
}
name, model, count, d, rate, raw = CFG[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
codec = P.make_codec(name)
vals, _ = H.gen_arrays(model, count, 65536, d, seed=1, rate_ppm=rate)
flat = vals.reshape(-1)
enc = H.encode_chunks(codec, flat, np.arange(count, dtype=np.uint64) * 65536,
                      np.full(count, 65536, np.uint32), allow_wrap=model == "geometric", raw=raw)
b = P.DeviceBatch(codec, enc, raw=raw)
for _ in range(reps):
    b.decode()
torch.cuda.synchronize()
b.check()
print("ok", b.algorithmic_bytes)
