"""BASELINE.json config shapes, encoded by the REFERENCE (oracle/_ref).

Each case holds inputs of one config's shape (smaller array counts), the
words the reference encoder produced for them — encode_array
(codec.cpp:14-37) for C1/C3/C5, the wrapping Codec::encode_deltas rule for
C4, Codec::encode_deltas per chunk for C2's raw sweep —
and the reference decoder's output on those words (decode_array /
decode_deltas).  The GPU must reproduce that output word for word on every
decode path (tests/test_gpu_configs.py); the harness encoder must reproduce
the reference's words (tests/test_config_words.py).

Run as a script (`python -m tests.config_cases`), it checks every case on
the GPU paths the current environment selects (IZG_SPLIT, IZG_GROUP,
IZG_BIG_IDX_BATCH are read once per process, so forced paths need a fresh
process) and prints "ok".
"""
from __future__ import annotations

import numpy as np

import harness as H

N = 65536
SEED = 777


def _arrays(model, count, d, seed, rate=0):
    vals, _ = H.gen_arrays(model, count, N, d, seed=seed, rate_ppm=rate)
    return vals


def _ref_array_case(ref, label, name, vals, wrap=False, threads=8):
    m = vals.shape[0]
    offs = np.arange(m, dtype=np.uint64) * N
    counts = np.full(m, N, dtype=np.uint32)
    words, table = ref.encode_batch(name, vals.reshape(-1), offs, counts, wrap=wrap,
                                    threads=threads)
    b = ref.batch_new(name)
    b.add(name, vals.reshape(-1), offs, counts, wrap=wrap, threads=threads)
    b.decode(threads=threads)
    ref_out = np.concatenate([b.output(i, N) for i in range(m)])
    b.close()
    return {"label": label, "name": name, "raw": False, "wrap": wrap, "values": vals,
            "words": words, "table": table, "ref_out": ref_out}


def c1(ref):
    """C1: SIMD-BP128+D4, ClusterData over [0, 2^29) (BASELINE recipe)."""
    return [_ref_array_case(ref, "C1", "simdbp128-s4", _arrays("cluster", 128, 29, SEED))]


def c2(ref):
    """C2: raw SIMD-BP128 (no delta), one 65,536-value chunk per b = 0..32,
    values uniform in [0, 2^b) (Codec::encode_deltas / decode_deltas)."""
    rng = np.random.default_rng(SEED)
    pays, vals = [], []
    for b in range(33):
        hi = 1 << b
        v = (rng.integers(0, hi, size=N, dtype=np.uint64) if b else np.zeros(N, np.uint64))
        v = v.astype(np.uint32)
        pays.append(ref.encode_deltas("simdbp128", v))
        vals.append(v)
    # placed like izg_layout_chunks (16-byte aligned payloads)
    table = np.zeros(33, dtype=H.CHUNK_DTYPE)
    pos = 0
    for i, p in enumerate(pays):
        pos = (pos + 3) // 4 * 4
        table[i] = (pos, len(p), N, i * N)
        pos += len(p)
    words = np.zeros((pos + 3) // 4 * 4 + 4, dtype=np.uint32)
    ref_out = []
    for t, p in zip(table, pays):
        words[int(t["word_off"]):int(t["word_off"]) + len(p)] = p
        out, used = ref.decode_deltas("simdbp128", p, N)
        assert used == len(p)
        ref_out.append(out)
    return [{"label": "C2", "name": "simdbp128", "raw": True, "wrap": False,
             "values": np.stack(vals), "words": words, "table": table,
             "ref_out": np.concatenate(ref_out)}]


def c3(ref):
    """C3: d in {18, 22, 26, 29} x {ClusterData, Uniform} x {D1, D4}."""
    cases = []
    for model in ("cluster", "uniform"):
        for d in (18, 22, 26, 29):
            vals = _arrays(model, 8, d, SEED + d)
            for name in ("simdbp128", "simdbp128-s4"):
                cases.append(_ref_array_case(ref, f"C3 {model} d={d}", name, vals))
    return cases


def c4(ref):
    """C4: SIMD-FastPFOR+D4, geometric(mean 8) gaps with 1/5/10% outliers
    (prefix sums wrap mod 2^32: the reference's wrapping encode)."""
    return [_ref_array_case(ref, f"C4 {ppm // 10000}%", "simdfastpfor-s4",
                            _arrays("geometric", 32, 32, SEED + ppm, rate=ppm), wrap=True)
            for ppm in (10000, 50000, 100000)]


def c5(ref):
    """C5: a 256-array sample, d ~ U{20..29} per array, both codecs."""
    vals = _arrays("cluster", 256, (20, 29), SEED)
    return [_ref_array_case(ref, "C5", name, vals)
            for name in ("simdbp128-s4", "simdfastpfor-s4")]


def all_cases(ref):
    return c1(ref) + c2(ref) + c3(ref) + c4(ref) + c5(ref)


def check_gpu(cases, paths=("fused", "ws", "host")):
    """Decode every case on the GPU through the C ABI and compare word for
    word with the reference's decode of the same words."""
    import paper_1209_2137_b200 as P

    for c in cases:
        codec = P.make_codec(c["name"])
        enc = P.Encoded(c["words"], c["table"])
        for path in paths:
            if path == "host":
                got, st = P.decode_array(codec, enc, raw=c["raw"], return_status=True)
                assert not st.any(), (c["label"], c["name"], path, st[st != 0][:4])
                got = got[:len(c["ref_out"])]
            else:
                b = P.DeviceBatch(codec, enc, raw=c["raw"], indexed=(path == "ws"))
                b.decode()
                st = b.statuses()
                assert not st.any(), (c["label"], c["name"], path, st[st != 0][:4])
                used = b.consumed[:b.n_chunks].cpu().numpy().astype(np.int64)
                assert np.array_equal(used, c["table"]["n_words"].astype(np.int64)), \
                    (c["label"], c["name"], path)
                got = b.output()
            if not np.array_equal(got, c["ref_out"]):
                bad = int(np.nonzero(got != c["ref_out"])[0][0])
                raise AssertionError(f"{c['label']} {c['name']} {path}: differs from the "
                                     f"reference at integer {bad}")


def main():
    from oracle.pyoracle import Reference

    check_gpu(all_cases(Reference()))
    print("ok")


if __name__ == "__main__":
    main()
