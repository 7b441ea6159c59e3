"""Decode throughput of the scalar-group codecs on
reference-encoded ClusterData (the product has no encoder for them; the
inputs come from the reference compiled into oracle/_ref).  CUDA events,
L2 flushed between repetitions."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P
from oracle.pyoracle import Reference
from paper_1209_2137_b200.device import host_checksum

ref = Reference()
count = int(os.environ.get("F3_ARRAYS", "1024"))
vals, _ = H.gen_arrays("cluster", count, 65536, (20, 29), seed=1)
flat = vals.reshape(-1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in sys.argv[1:] or ["bp32-s4", "fastpfor-s4", "simplepfor-s4", "simdbp128-s4",
                             "simdfastpfor-s4"]:
    codec = P.make_codec(name)
    payloads, counts = [], []
    for row in vals:
        for n, p in ref.encode_array(name, row):
            payloads.append(p)
            counts.append(n)
    enc = P.layout(codec, payloads, counts)
    b = P.DeviceBatch(codec, enc)
    for _ in range(3):
        b.decode()
    torch.cuda.synchronize()
    b.check()
    ok = b.checksum() == host_checksum(flat)
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.decode(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = float(np.median(ts))
    gb = b.algorithmic_bytes / t / 1e9
    print(json.dumps(dict(name=name, arrays=count, ok=bool(ok),
                          bits_per_int=round(32 * b.payload_words / flat.size, 3),
                          ms=round(t * 1e3, 4), gints=round(flat.size / t / 1e9, 1),
                          alg_GBps=round(gb, 1), frac=round(gb / 6532.9, 3))), flush=True)
