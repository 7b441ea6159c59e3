"""Decode a small batch (for ncu launch lists): CHUNKS arrays of 65,536.
    python tools/profile_small.py <simdbp128-s4|simdfastpfor-s4> <chunks> [reps]
IZG_NOWS=1: no workspace (izg_decode: SIMD-BP128 small batches take the group
kernel instead of the split kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import harness as H
import paper_1209_2137_b200 as P

name, count = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
codec = P.make_codec(name)
geo = "fastpfor" in name
vals, _ = H.gen_arrays("geometric" if geo else "cluster", count, 65536, 32 if geo else 29,
                       seed=1, rate_ppm=100000 if geo else 0)
enc = H.encode_chunks(codec, vals.reshape(-1), np.arange(count, dtype=np.uint64) * 65536,
                      np.full(count, 65536, np.uint32), allow_wrap=geo)
b = P.DeviceBatch(codec, enc, indexed=os.environ.get("IZG_NOWS") != "1")
for _ in range(reps):
    b.decode()
torch.cuda.synchronize()
b.check()
print("ok")
