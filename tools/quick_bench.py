"""Developer timing loop: decode throughput of one config (CUDA events)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P

try:  # the driver-measured copy bandwidth (roofline denominator)
    PEAK = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                             "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    PEAK = 6532.9

def run(name, model, count, d, seed=1, rate=0, reps=20, raw=False):
    codec = P.make_codec(name)
    t0 = time.time()
    vals, _ = H.gen_arrays(model, count, 65536, d, seed=seed, rate_ppm=rate)
    flat = vals.reshape(-1)
    offs = np.arange(count, dtype=np.uint64) * 65536
    enc = H.encode_chunks(codec, flat, offs, np.full(count, 65536, np.uint32),
                          allow_wrap=(model == "geometric"), raw=raw)
    t1 = time.time()
    b = P.DeviceBatch(codec, enc, raw=raw, indexed=os.environ.get("IZG_FUSED") != "1")
    for _ in range(3): b.decode()
    torch.cuda.synchronize(); b.check()
    if not raw:
        from paper_1209_2137_b200.device import host_checksum
        ok = b.checksum() == host_checksum(flat)
    else:
        ok = np.array_equal(b.output()[:65536*4], flat[:65536*4])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.decode(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = float(np.median(ts))
    n = count * 65536
    gb = b.algorithmic_bytes / t / 1e9
    print(json.dumps(dict(name=name, model=model, d=d, rate=rate, raw=raw, ok=bool(ok),
        bits_per_int=round(32 * b.payload_words / n, 3), ms=round(t * 1e3, 4),
        gints=round(n / t / 1e9, 2), alg_GBps=round(gb, 1), frac=round(gb / PEAK, 3),
        prep_s=round(t1 - t0, 1))), flush=True)

if __name__ == "__main__":
    which = sys.argv[1:] or ["c1"]
    for w in which:
        if w == "c1": run("simdbp128-s4", "cluster", 1024, 29)
        if w == "c1big": run("simdbp128-s4", "cluster", 8192, 29)
        if w == "d1": run("simdbp128", "cluster", 4096, 29)
        if w == "d4u": run("simdbp128-s4", "uniform", 4096, 26)
        if w == "c4": run("simdfastpfor-s4", "geometric", 2048, 32, rate=100000)
        if w == "c4_1": run("simdfastpfor-s4", "geometric", 2048, 32, rate=10000)
        if w == "c5fp": run("simdfastpfor-s4", "cluster", 8192, (20, 29))
        if w == "c5bp": run("simdbp128-s4", "cluster", 8192, (20, 29))
        if w == "c5fpbig": run("simdfastpfor-s4", "cluster", 32768, (20, 29), reps=8)
        if w == "fp29": run("simdfastpfor-s4", "cluster", 8192, 29)
        if w == "raw":
            for b in (0, 8, 16, 24, 32): run("simdbp128", "raw", 4096, b, raw=True)


def run_encode(name, model, count, d, rate=0, reps=10):
    """GPU encoder throughput (izg_encode) on device-resident values."""
    import paper_1209_2137_b200._native as N
    codec = P.make_codec(name)
    vals, _ = H.gen_arrays(model, count, 65536, d, seed=3, rate_ppm=rate)
    flat = vals.reshape(-1)
    L = N.lib()
    counts = np.full(count, 65536, np.uint32)
    bound = (L.izg_encode_bound(codec.codec, 65536) + 3) // 4 * 4
    table = np.zeros(count, dtype=N.CHUNK_DTYPE)
    table["word_off"] = np.arange(count, dtype=np.uint64) * bound
    table["n"] = counts
    table["out_off"] = np.arange(count, dtype=np.uint64) * 65536
    dv = torch.from_numpy(flat.view(np.int32)).cuda()
    dt = torch.from_numpy(table.view(np.uint8)).cuda()
    dw = torch.zeros(count * bound + 4, dtype=torch.int32, device="cuda")
    ds = torch.zeros(count, dtype=torch.int32, device="cuda")
    wrap = int(model == "geometric")
    def go():
        rc = L.izg_encode(codec.codec, codec.delta, dv.data_ptr(), dt.data_ptr(), count, dw.data_ptr(),
                          ds.data_ptr(), wrap, torch.cuda.current_stream().cuda_stream)
        assert rc == 0
    for _ in range(3): go()
    torch.cuda.synchronize()
    assert int(ds.abs().sum()) == 0
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); go(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = float(np.median(ts))
    print(json.dumps(dict(encode=name, model=model, gints=round(flat.size / t / 1e9, 2), ms=round(t * 1e3, 3))), flush=True)


if __name__ == "__main__" and "enc" in sys.argv[1:]:
    run_encode("simdbp128-s4", "cluster", 4096, (20, 29))
    run_encode("simdfastpfor-s4", "cluster", 4096, (20, 29))
    run_encode("simdfastpfor-s4", "geometric", 2048, 32, rate=100000)
