"""Developer: randomized stress of the SIMD-BP128 relay kernel (csrc/relay.cuh)
against the one-warp kernel: random batch sizes inside its default range
(2,432..14,208 chunks; or any size with IZG_RELAY=1), ragged lengths with VByte
remainders, every delta mode and the raw mode, random bit flips and truncated
payloads; statuses, words consumed and the output of every chunk that decodes
must be identical, over repeated launches of each batch.

    [IZG_RELAY=1 IZG_RELAY_SEGS=..] python tools/relay_stress.py [seconds] [seed]
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P
from paper_1209_2137_b200.codec import Encoded

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
forced = os.environ.get("IZG_RELAY") == "1"
t_end = time.time() + budget
rounds = chunks = corrupted = 0
while time.time() < t_end:
    raw = rng.random() < 0.2
    name = "simdbp128" if raw else str(rng.choice(["simdbp128-s4", "simdbp128", "simdbp128-d2", "simdbp128-dm"]))
    codec = P.make_codec(name)
    count = int(rng.choice([3, 40, 700, 2000])) if forced and rng.random() < 0.5 else int(rng.integers(2432, 14209))
    big = rng.random(count) < rng.choice([0.02, 0.2, 0.6])
    lens = np.where(big, 65536, rng.integers(1, 9000, size=count)).astype(np.uint32)
    if raw:
        lens = np.maximum(128, lens // 128 * 128).astype(np.uint32)
    offs = np.concatenate([[0], np.cumsum(lens, dtype=np.uint64)[:-1]]).astype(np.uint64)
    total = int(lens.sum())
    bits = int(rng.integers(1, 16))  # 65,536 gaps below 2^16 stay under 2^32
    gaps = rng.integers(0, 1 << bits, size=total, dtype=np.uint32)
    if raw:
        flat = gaps
    else:
        flat = np.cumsum(gaps, dtype=np.uint64)
        base = np.repeat(np.concatenate([[0], flat[offs[1:] - 1]]).astype(np.uint64), lens)
        flat = ((flat - base) & 0xFFFFFFFF).astype(np.uint32)   # restart per array; < 2^32 for these sizes
    enc = H.encode_chunks(codec, flat, offs, lens, raw=raw)
    w = enc.words.copy()
    nbad = int(rng.choice([0, 0, 5, 200]))
    for c in rng.integers(0, count, size=nbad):
        off, nw = int(enc.table["word_off"][c]), int(enc.table["n_words"][c])
        if nw:
            w[off + int(rng.integers(0, nw))] ^= np.uint32(1) << np.uint32(rng.integers(0, 32))
    table = enc.table.copy()
    for c in rng.integers(0, count, size=nbad // 4):   # truncated payloads
        if table["n_words"][c] > 1:
            table["n_words"][c] = int(rng.integers(0, int(table["n_words"][c])))
    bad = Encoded(w, table)
    a = P.DeviceBatch(codec, bad, raw=raw, relay_long_only=False)
    b = P.DeviceBatch(codec, bad, raw=raw, indexed=False)
    assert a.workspace is not None, count
    b.decode(); torch.cuda.synchronize()
    sb, ob = b.statuses(), b.output()
    cb = b.consumed[:count].cpu().numpy()
    if nbad == 0:
        assert not sb.any() and np.array_equal(ob[:total], flat), ("one-warp baseline", name, count)
    good = np.repeat(sb == 0, lens)
    for rep in range(2):
        a.out.fill_(0)
        a.decode(); torch.cuda.synchronize()
        sa = a.statuses()
        if not np.array_equal(sa, sb):
            i = int(np.nonzero(sa != sb)[0][0])
            raise SystemExit(f"STATUS MISMATCH {name} raw={raw} count={count} chunk={i} relay={sa[i]} one-warp={sb[i]} n={lens[i]}")
        if not np.array_equal(a.consumed[:count].cpu().numpy(), cb):
            raise SystemExit(f"CONSUMED MISMATCH {name} raw={raw} count={count}")
        oa = a.output()
        if not np.array_equal(oa[:total][good], ob[:total][good]):
            raise SystemExit(f"OUTPUT MISMATCH {name} raw={raw} count={count} rep={rep}")
    rounds += 1
    chunks += count
    corrupted += int((sb != 0).sum())
    del a, b
    torch.cuda.empty_cache()
print(f"ok: {rounds} batches, {chunks} chunks, {corrupted} rejected chunks, forced={forced}")
