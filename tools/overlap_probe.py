"""Developer: the C5 step with SIMD-FastPFOR's page index pass on a second
stream, concurrent with the SIMD-BP128 decode (izg_decode_ws_phase), against
the serial step.  IZG_BP_MAX_CTAS caps the persistent SIMD-BP128 decode grid so
the index pass's CTAs can co-reside."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P

count = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
vals, _ = H.gen_arrays("cluster", count, 65536, (20, 29), seed=1)
flat = vals.reshape(-1)
offs = np.arange(count, dtype=np.uint64) * 65536
cnt = np.full(count, 65536, np.uint32)
out = torch.empty(count * 65536, dtype=torch.int32, device="cuda")
bp = P.DeviceBatch(P.make_codec("simdbp128-s4"), H.encode_chunks("simdbp128-s4", flat, offs, cnt), out=out)
fp = P.DeviceBatch(P.make_codec("simdfastpfor-s4"), H.encode_chunks("simdfastpfor-s4", flat, offs, cnt), out=out)
s1 = torch.cuda.current_stream()
s2 = torch.cuda.Stream()

def serial():
    bp.decode(s1); fp.decode(s1)

def overlap():
    ev = torch.cuda.Event()
    ev.record(s1)
    s2.wait_event(ev)
    fp.decode_phase(1, s2)
    bp.decode(s1)
    e2 = torch.cuda.Event()
    e2.record(s2)
    s1.wait_event(e2)
    fp.decode_phase(2, s1)

def timeit(f, reps=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s1); f(); b.record(s1); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))

from paper_1209_2137_b200.device import host_checksum
for name, f in (("serial", serial), ("overlap", overlap)):
    ms = timeit(f)
    fp.check(); ok = fp.checksum() == host_checksum(flat)
    print(json.dumps({"mode": name, "cap": os.environ.get("IZG_BP_MAX_CTAS"), "ms": round(ms, 4), "ok": ok}), flush=True)
