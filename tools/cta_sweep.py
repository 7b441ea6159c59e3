"""Developer sweep: SIMD-BP128+D4 decode time by batch size, for the path
izg_decode_ws picks (DeviceBatch default) — run once with IZG_CTA=1 and once
with IZG_CTA=0 to place the CTA kernel's thresholds."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P

codec = P.make_codec(sys.argv[1] if len(sys.argv) > 1 else "simdbp128-s4")
counts = [int(x) for x in os.environ.get("COUNTS", "64,128,256,384,512,768,1024,1536,2048,3072,4096").split(",")]
vals, _ = H.gen_arrays("cluster", max(counts), 65536, 29, seed=1)
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
    ok = np.array_equal(b.output()[:65536 * 2], flat[:65536 * 2])
    print(json.dumps({"cta": os.environ.get("IZG_CTA"), "tail": os.environ.get("IZG_CTA_TAIL"), "chunks": count, "ms": round(float(np.median(ts)), 4),
                      "ok": bool(ok)}), flush=True)
