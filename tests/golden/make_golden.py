"""Regenerate tests/golden/ref_vectors.npz from the REFERENCE library
(oracle/_ref, compiled from /root/reference/proj/core/src by oracle/Makefile).

    python tests/golden/make_golden.py

Every payload, decoded array and error status in the fixture was produced by
the reference's own encode_array / encode_deltas / decode_array; nothing here
comes from this repository's encoder or decoder.  The fixture travels with the
repo, so the parity tests need no reference tree at run time.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import RefError, Reference  # noqa: E402
from tests.test_oracle_vs_ref import WHAT  # noqa: E402

NAMES = ["simdbp128", "simdbp128-s4", "simdfastpfor", "simdfastpfor-s4"]


def random_sorted(rng, n, max_delta):
    d = rng.integers(0, max_delta + 1, size=n, dtype=np.uint64)
    return np.minimum(np.cumsum(d), 0xFFFFFFFF).astype(np.uint32)


def main():
    ref = Reference()
    rng = np.random.default_rng(20120910)
    out = {}
    # encode_array / decode_array vectors
    for name in NAMES:
        sizes = [1, 130, 2049 + 5, 65536 + 77] if name.endswith("-s4") else [129, 4096 + 3]
        for k, n in enumerate(sizes):
            vals = random_sorted(rng, n, int(rng.choice([40, 3000, 1 << 20])))
            if k == 2:  # outliers for the patched codec
                gaps = np.diff(vals, prepend=0).astype(np.uint64)
                gaps[::23] += rng.integers(1 << 12, 1 << 20, size=len(gaps[::23]), dtype=np.uint64)
                vals = np.minimum(np.cumsum(gaps), 0xFFFFFFFF).astype(np.uint32)
            chunks = ref.encode_array(name, vals)
            assert np.array_equal(ref.decode_array(name, chunks), vals)
            key = f"arr/{name}/{k}"
            out[key + "/values"] = vals
            out[key + "/lens"] = np.array([c for c, _ in chunks], np.uint32)
            out[key + "/payload"] = np.concatenate([p for _, p in chunks])
            out[key + "/nwords"] = np.array([len(p) for _, p in chunks], np.uint32)
    # decode_deltas at every width
    for codec in ("simdbp128", "simdfastpfor"):
        for b in range(33):
            n = 128 * (1 + b % 5)
            v = (rng.integers(0, 2**32, size=n, dtype=np.uint64) & ((1 << b) - 1)).astype(np.uint32)
            if codec == "simdfastpfor" and b < 30:
                v[::17] |= np.uint32(1 << (b + 2))
            out[f"raw/{codec}/{b}/values"] = v
            out[f"raw/{codec}/{b}/payload"] = ref.encode_deltas(codec, v)
    # corrupted chunks and the reference's verdict
    for name in NAMES:
        vals = random_sorted(rng, 1500, 4000)
        payload = ref.encode_array(name, vals)[0][1]
        pays, stats, decs = [], [], []
        for rep in range(60):
            p = payload.copy()
            bb = p.view(np.uint8)
            for _ in range(1 + rep % 3):
                bb[rng.integers(0, len(bb))] = rng.integers(0, 256)
            if rep % 7 == 0:
                p = p[:int(rng.integers(0, len(p)))]
            try:
                dec = ref.decode_array(name, [(1500, p)])
                st = 0
            except RefError as e:
                st, dec = WHAT[e.what], np.zeros(1500, np.uint32)
            pays.append(p)
            stats.append(st)
            decs.append(dec)
        out[f"bad/{name}/payload"] = np.concatenate(pays)
        out[f"bad/{name}/nwords"] = np.array([len(p) for p in pays], np.uint32)
        out[f"bad/{name}/status"] = np.array(stats, np.int32)
        out[f"bad/{name}/decoded"] = np.stack(decs)
    # an INTZPK01 container written by the reference (container.cpp:112-130)
    # and the chunk table its reader returns (container.cpp:132-169)
    crng = np.random.default_rng(20240)
    arrays = [random_sorted(crng, n, 3000) for n in (0, 7, 129, 70000)]
    data = ref.container_write_encoded("simdbp128-s4", arrays)
    _, rarr = ref.container_read_encoded(data)
    out["container_bytes"] = np.frombuffer(data, dtype=np.uint8)
    out["container_n"] = np.array([n for a in rarr for n, _ in a], np.uint32)
    out["container_n_words"] = np.array([len(p) for a in rarr for _, p in a], np.uint32)
    out["container_values"] = np.concatenate(arrays)
    np.savez_compressed(os.path.join(HERE, "ref_vectors.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
