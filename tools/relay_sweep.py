"""Developer sweep: SIMD-BP128 decode time by batch size for the path
izg_decode_ws picks (DeviceBatch default) — run with IZG_RELAY=0 and with
IZG_RELAY=1 IZG_RELAY_SEGS=2/4/8/16 to place the relay kernel's thresholds
(csrc/relay.cuh).  COUNTS, MODEL (cluster/uniform), D, codec name as argv[1].
Every batch is verified by the order-sensitive checksum of its input."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P
from paper_1209_2137_b200.device import host_checksum

name = sys.argv[1] if len(sys.argv) > 1 else "simdbp128-s4"
codec = P.make_codec(name)
counts = [int(x) for x in os.environ.get("COUNTS", "3552,4096,6144,8192,12288,16384").split(",")]
model, d = os.environ.get("MODEL", "cluster"), int(os.environ.get("D", "29"))
vals, _ = H.gen_arrays(model, max(counts), 65536, d, seed=1)
flat = vals.reshape(-1)
for count in counts:
    enc = H.encode_chunks(codec, flat[:count * 65536], np.arange(count, dtype=np.uint64) * 65536,
                          np.full(count, 65536, np.uint32))
    b = P.DeviceBatch(codec, enc)
    for _ in range(3):
        b.decode()
    torch.cuda.synchronize()
    b.check()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(15):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.decode(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ok = b.checksum() == host_checksum(flat[:count * 65536])
    t = float(np.median(ts))
    print(json.dumps({"relay": os.environ.get("IZG_RELAY"), "segs": os.environ.get("IZG_RELAY_SEGS"),
                      "codec": name, "model": model, "d": d, "chunks": count, "ms": round(t, 4),
                      "GBps": round(b.algorithmic_bytes / t / 1e6, 1), "ok": bool(ok)}), flush=True)
    del b
    torch.cuda.empty_cache()
