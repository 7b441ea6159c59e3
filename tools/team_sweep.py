"""Developer: SIMD-FastPFOR decode time by batch size (izg_decode_ws), for the
dispatch thresholds of the team kernel: run once with IZG_TEAM=0 (split /
one warp per page / large-batch shape) and once with IZG_TEAM=1.

    IZG_TEAM=0 python tools/team_sweep.py [c5|c4] ; IZG_TEAM=1 python tools/team_sweep.py [c5|c4]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P

which = sys.argv[1] if len(sys.argv) > 1 else "c5"
model, d, rate = ("cluster", (20, 29), 0) if which == "c5" else ("geometric", 32, 100000)
counts = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else \
    [16, 64, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768]
codec = P.make_codec("simdfastpfor-s4")
nmax = max(counts)
vals, _ = H.gen_arrays(model, nmax, 65536, d, seed=1, rate_ppm=rate)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for count in counts:
    flat = vals[:count].reshape(-1)
    enc = H.encode_chunks(codec, flat, np.arange(count, dtype=np.uint64) * 65536,
                          np.full(count, 65536, np.uint32), allow_wrap=model == "geometric")
    b = P.DeviceBatch(codec, enc)
    for _ in range(3): b.decode()
    torch.cuda.synchronize(); b.check()
    from paper_1209_2137_b200.device import host_checksum
    ok = b.checksum() == host_checksum(flat)
    ts = []
    for _ in range(15 if count <= 8192 else 6):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.decode(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps(dict(cfg=which, team=os.environ.get("IZG_TEAM"), split=os.environ.get("IZG_SPLIT"),
                          pages=count, ms=round(float(np.median(ts)), 4), ok=bool(ok))), flush=True)
    del b
