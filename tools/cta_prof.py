"""Developer: time split of the CTA kernel's consumer units (IZG_CTA_PROF build)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P
L = P._native.lib()
count = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
codec = P.make_codec("simdbp128-s4")
vals, _ = H.gen_arrays("cluster", count, 65536, 29, seed=1)
enc = H.encode_chunks(codec, vals.reshape(-1), np.arange(count, dtype=np.uint64) * 65536,
                      np.full(count, 65536, np.uint32))
b = P.DeviceBatch(codec, enc)
b.decode(); torch.cuda.synchronize(); b.check()
buf = np.zeros((160, 17, 8), np.uint64)
L.izg_debug_cta_prof(buf.ctypes.data, buf.nbytes, 1)
b.decode(); torch.cuda.synchronize()
L.izg_debug_cta_prof(buf.ctypes.data, buf.nbytes, 0)
names = ["find chunk", "walk wait", "piece wait", "unpack+scan", "carry wait", "post+stores"]
cons = [w for w in range(17) if w % 4]
tot = buf[:148, cons, :6].sum(axis=(0, 1)).astype(np.float64)
units = count * 64
print("cycles per unit (avg over units):", {n: round(t / units) for n, t in zip(names, tot)})
print("sum", round(tot.sum() / units))
pr = buf[:148, 0, 6:8].sum(axis=0).astype(np.float64)
print("producer cycles per chunk: landing waits", round(pr[0] / count), "no-progress sleeps", round(pr[1] / count))

tr = np.zeros((64, 6), np.int64)
L.izg_debug_cta_trace(tr.ctypes.data)
t0 = tr[0, 0]
print("CTA 0 per chunk (cycles from first claim): claim, published, walk done, first unit, done")
for i in range(min(20, 64)):
    print(i, *(int(x - t0) if x else 0 for x in tr[i, :5]))
