"""SURVEY.md §8 f4 measurement: decode two posting lists and intersect them on
the GPU, (a) device-resident (CUDA events) and (b) end to end from pinned host
compressed buffers (H2D of the compressed words, D2H of the intersection
only), beside a single-threaded numpy binary-search intersection of the
already-decoded host arrays.  The device number is given for both the
unfused path (decode both, izg_intersect_sorted) and the fused one (decode
the short list, izg_decode_intersect for the long one); e2e uses the fused
path.  CODEC=<name> picks the codec (default simdbp128-s4)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P

na, nb = int(os.environ.get("NA", 1 << 26)), int(os.environ.get("NB", 1 << 22))
rng = np.random.default_rng(1)
a = np.cumsum(rng.integers(1, 40, size=na, dtype=np.uint64)).astype(np.uint32)
pick = rng.random(na) < (nb / na) * 0.5
b = np.unique(np.concatenate([a[pick], np.cumsum(rng.integers(1, 40 * na // nb, size=nb // 2, dtype=np.uint64)).astype(np.uint32)])).astype(np.uint32)
codec = P.make_codec(os.environ.get("CODEC", "simdbp128-s4"))
ea, eb = H.encode_array(codec, a), H.encode_array(codec, b)
want = np.intersect1d(a, b)
def cpu_isect(a, b):  # sorted inputs: binary-search the shorter in the longer (the GPU's algorithm)
    s, l = (a, b) if len(a) <= len(b) else (b, a)
    s = s[np.concatenate([[True], s[1:] != s[:-1]])]
    i = np.searchsorted(l, s)
    ok = i < len(l)
    ok[ok] = l[i[ok]] == s[ok]
    return s[ok]
assert np.array_equal(cpu_isect(a, b), want)
t = time.perf_counter(); cpu_isect(a, b); t_np = time.perf_counter() - t

ba, bb = P.DeviceBatch(codec, ea), P.DeviceBatch(codec, eb)
def dev_step():
    ba.decode(); bb.decode()
    return P.intersect_device(ba.out[:ba.n_out], bb.out[:bb.n_out])
r = dev_step(); torch.cuda.synchronize()
assert np.array_equal(r.cpu().numpy().view(np.uint32), want)
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dev_step(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
t_dev = float(np.median(ts))

# fused: the short list decoded to HBM, the long one decoded and probed in
# shared memory (izg_decode_intersect), never written
bl = P.DeviceBatch(codec, ea, materialize=False, indexed=False)
def fused_step():
    bb.decode()
    return P.decode_intersect_device(bl, bb.out[:bb.n_out])
r = fused_step(); torch.cuda.synchronize()
assert np.array_equal(r.cpu().numpy().view(np.uint32), want)
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fused_step(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
t_fused = float(np.median(ts))

# end to end: pinned compressed words in, intersection out
hw = [torch.from_numpy(e.words.view(np.int32)).pin_memory() for e in (ea, eb)]
dw = [torch.empty_like(h, device="cuda") for h in hw]
def e2e_step():
    for h, d in zip(hw, dw):
        d.copy_(h, non_blocking=True)
    bl.words, bb.words = dw
    r = fused_step()
    return r.cpu()
e2e_step()
t = time.perf_counter()
for _ in range(5):
    out = e2e_step()
t_e2e = (time.perf_counter() - t) / 5
assert np.array_equal(out.numpy().view(np.uint32), want)
n = na + len(b)
print(json.dumps(dict(codec=codec.name, na=na, nb=len(b), common=len(want), device_ms=round(t_dev * 1e3, 3),
                      device_Gints=round(n / t_dev / 1e9, 1),
                      fused_ms=round(t_fused * 1e3, 3), fused_Gints=round(n / t_fused / 1e9, 1), e2e_ms=round(t_e2e * 1e3, 2),
                      e2e_Gints=round(n / t_e2e / 1e9, 1), numpy_searchsorted_1thread_ms=round(t_np * 1e3, 1),
                      h2d_bytes=int(sum(e.words.nbytes for e in (ea, eb))),
                      d2h_bytes=int(4 * len(want)))))
