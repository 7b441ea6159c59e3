"""Developer: where a page's time goes in the team SIMD-FastPFOR decode
(IZG_TEAM_PROF build: python tools/build_variant.py tprof -DIZG_TEAM_PROF;
IZG_TEAM=1 IZG_SPLIT=0 IZG_LIB_PATH=.../variants/tprof.so python tools/team_prof.py [c5fp|c4])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P
L = P._native.lib()
which = sys.argv[1] if len(sys.argv) > 1 else "c5fp"
model, count, d, rate = {"c5fp": ("cluster", 8192, (20, 29), 0), "c4": ("geometric", 2048, 32, 100000),
                         "fp29": ("cluster", 8192, 29, 0)}[which]
codec = P.make_codec("simdfastpfor-s4")
vals, _ = H.gen_arrays(model, count, 65536, d, seed=1, rate_ppm=rate)
enc = H.encode_chunks(codec, vals.reshape(-1), np.arange(count, dtype=np.uint64) * 65536,
                      np.full(count, 65536, np.uint32), allow_wrap=model == "geometric")
b = P.DeviceBatch(codec, enc)
b.decode(); torch.cuda.synchronize(); b.check()
buf = np.zeros(8, np.uint64)
L.izg_debug_team_prof(buf.ctypes.data, 1)
b.decode(); torch.cuda.synchronize()
L.izg_debug_team_prof(buf.ctypes.data, 0)
n = float(buf[0])
names = ["warp 0 waits: page descriptor", "warp 0 waits: exception window", "warp 0 waits: staged data",
         "warp 0 waits: carry mailbox", "warp 0: whole page", "staging warp: idle passes",
         "staging warp: cycles in unpack passes"]
for nm, v in zip(names, buf[1:]):
    print(f"{nm:40s} {float(v) / n:10.0f} per page")
