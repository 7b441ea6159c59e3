"""Developer: SIMD-BP128+D4 batches of SHORT chunks in the relay kernel's default range
(run with IZG_RELAY=0 and unset): the relay's levels past a short chunk's last segment
are claimed and skipped, which must not cost more than it gains elsewhere."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P
codec = P.make_codec("simdbp128-s4")
rng = np.random.default_rng(3)
for count in (2500, 4096, 14000):
    for n in (100, 1000, 8192, 20000):
        lens = np.full(count, n, np.uint32)
        offs = np.arange(count, dtype=np.uint64) * n
        flat = np.cumsum(rng.integers(0, 64, size=(count, n), dtype=np.uint32), axis=1, dtype=np.uint32).reshape(-1)
        enc = H.encode_chunks(codec, flat, offs, lens)
        b = P.DeviceBatch(codec, enc, relay_long_only=False)
        for _ in range(3):
            b.decode()
        torch.cuda.synchronize(); b.check()
        ts = []
        for _ in range(30):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); b.decode(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ok = np.array_equal(b.output(), flat)
        print(json.dumps({"relay": os.environ.get("IZG_RELAY"), "chunks": count, "ints": n,
                          "us": round(float(np.median(ts)) * 1e3, 1), "ok": bool(ok)}), flush=True)
