"""Launch one f3 codec's decode a few times (reference-encoded inputs; for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P
from oracle.pyoracle import Reference
name = sys.argv[1]
count = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
ref = Reference()
vals, _ = H.gen_arrays("cluster", count, 65536, (20, 29), seed=1)
codec = P.make_codec(name)
payloads, counts = [], []
for row in vals:
    for n, p in ref.encode_array(name, row):
        payloads.append(p); counts.append(n)
b = P.DeviceBatch(codec, P.layout(codec, payloads, counts))
for _ in range(3):
    b.decode()
torch.cuda.synchronize(); b.check(); print("ok")
