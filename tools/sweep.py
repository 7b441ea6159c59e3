"""BASELINE.json configs[1] and configs[2] measured on one GPU (JSON lines).

    python tools/sweep.py c2   # raw SIMD-BP128 unpack, b = 0..32, 2^28 values each
    python tools/sweep.py c3   # SIMD-BP128 delta variants D1/D2/D4/DM, 4096 x 65536,
                               # d in {18,22,26,29}, ClusterData and Uniform

Device-resident inputs, CUDA events around each decode launch, median of 20
after 3 warm-ups; a 256 MiB buffer is zeroed between launches (inputs plus
outputs exceed L2 anyway).  Every config is verified: C2 output against the
values, C3 by the order-sensitive checksum of the original arrays.
Roofline bytes = 4 * payload words + 4 per decoded integer;
peak = MEASURED_PEAKS.json hbm_gbs when present, else 6532.9 GB/s.
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P
from paper_1209_2137_b200.device import host_checksum

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6532.9


def timed(b, reps=20):
    for _ in range(3):
        b.decode()
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.decode(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return float(np.median(ts))


def run(name, model, count, d, raw, PK):
    codec = P.make_codec(name)
    vals, _ = H.gen_arrays(model, count, 65536, d, seed=11)
    flat = vals.reshape(-1)
    enc = H.encode_chunks(codec, flat, np.arange(count, dtype=np.uint64) * 65536,
                          np.full(count, 65536, np.uint32), raw=raw)
    b = P.DeviceBatch(codec, enc, raw=raw)
    t = timed(b)
    b.check()
    ok = (np.array_equal(b.output(), flat) if raw else b.checksum() == host_checksum(flat))
    n = count * 65536
    gbs = b.algorithmic_bytes / t / 1e9
    line = dict(config="c2" if raw else "c3", codec=name, model=model, d=d, arrays=count,
                ok=bool(ok), bits_per_int=round(32 * b.payload_words / n, 3),
                ms=round(t * 1e3, 4), gints=round(n / t / 1e9, 1), alg_GBps=round(gbs, 1),
                frac=round(gbs / PK, 3))
    print(json.dumps(line), flush=True)
    del b
    torch.cuda.empty_cache()


if __name__ == "__main__":
    PK = peak()
    for which in sys.argv[1:] or ["c2", "c3"]:
        if which == "c2":
            for bw in range(33):
                run("simdbp128", "raw", 4096, bw, True, PK)
        if which == "c3":
            for model in ("cluster", "uniform"):
                for d in (18, 22, 26, 29):
                    for name in ("simdbp128", "simdbp128-d2", "simdbp128-s4", "simdbp128-dm"):
                        run(name, model, 4096, d, False, PK)
