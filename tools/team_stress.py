"""Developer: randomized stress of the SIMD-FastPFOR workspace path (page index
pass + team decode) against the generated arrays: random batch sizes, array
lengths (ragged, with VByte remainders), outlier rates, data models, delta
modes and placements, repeated decodes of each batch under load.

    [IZG_INDEX_LANES_MIN=0] python tools/team_stress.py [seconds] [seed]
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
t_end = time.time() + budget
rounds = arrays = 0
while time.time() < t_end:
    name = str(rng.choice(["simdfastpfor-s4", "simdfastpfor", "simdfastpfor-d2", "simdfastpfor-dm"]))
    codec = P.make_codec(name)
    model = str(rng.choice(["cluster", "uniform", "geometric"]))
    count = int(rng.choice([1, 3, 17, 130, 400, 1500, 4000]))
    rate = int(rng.choice([0, 1000, 50000, 300000])) if model == "geometric" else 0
    d = 32 if model == "geometric" else int(rng.integers(18, 30))
    vals, _ = H.gen_arrays(model, count, 65536, d, seed=int(rng.integers(1, 1 << 30)), rate_ppm=rate)
    # ragged lengths: whole pages, short pages, lengths with a VByte remainder
    lens = np.where(rng.random(count) < 0.5, 65536,
                    rng.integers(1, 65537, size=count)).astype(np.uint32)
    offs = np.arange(count, dtype=np.uint64) * 65536
    flat = vals.reshape(-1)
    enc = H.encode_chunks(codec, flat, offs, lens, allow_wrap=model == "geometric")
    b = P.DeviceBatch(codec, enc)
    for rep in range(3):
        b.out.zero_()
        b.decode()
        torch.cuda.synchronize()
        st = b.statuses()
        assert not st.any(), (name, model, count, rate, st[st != 0][:4])
        got = b.out.cpu().numpy().view(np.uint32)
        for t, o, n in zip(enc.table, offs, lens):
            g = got[int(t["out_off"]):int(t["out_off"]) + int(n)]
            w = flat[int(o):int(o) + int(n)]
            if not np.array_equal(g, w):
                bad = np.nonzero(g != w)[0]
                raise SystemExit(f"MISMATCH {name} {model} count={count} rate={rate} d={d} rep={rep} "
                                 f"n={n} first={bad[:4]} of {len(bad)}")
    rounds += 1
    arrays += count
print(f"ok: {rounds} batches, {arrays} arrays")
