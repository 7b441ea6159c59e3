"""Split (several warps per chunk) vs one-warp-per-chunk decode across batch
sizes: CUDA-event time of DeviceBatch.decode() with the workspace (split
below the threshold) and without (izg_decode, one warp per chunk).

    IZG_SPLIT=1 python tools/split_sweep.py     # force split for every size
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import harness as H
import paper_1209_2137_b200 as P


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, model, d, rate in [("simdbp128-s4", "cluster", 29, 0),
                             ("simdfastpfor-s4", "geometric", 32, 100000)]:
    codec = P.make_codec(name)
    for count in [64, 128, 256, 512, 1024, 2048, 4096]:
        vals, _ = H.gen_arrays(model, count, 65536, d, seed=1, rate_ppm=rate)
        flat = vals.reshape(-1)
        enc = H.encode_chunks(codec, flat, np.arange(count, dtype=np.uint64) * 65536,
                              np.full(count, 65536, np.uint32), allow_wrap=model == "geometric")
        ws = P.DeviceBatch(codec, enc)
        one = P.DeviceBatch(codec, enc, indexed=False, out=ws.out)
        t_ws = timed(ws.decode)
        ws.check()
        ok = np.array_equal(ws.output(), flat)
        t_one = timed(one.decode)
        print(json.dumps(dict(codec=name, chunks=count, ws_ms=round(t_ws, 4),
                              one_warp_ms=round(t_one, 4), ws_path_ok=bool(ok),
                              split=bool(ws.workspace is not None and (codec.codec == 0 or
                                  ws.workspace.numel() > count * (16 + 128 + 512 * 16))))))
