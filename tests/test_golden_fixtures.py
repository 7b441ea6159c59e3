"""Committed reference vectors (tests/golden/ref_vectors.npz, produced by the
reference library itself via tests/golden/make_golden.py) against the oracle,
the host encoder, and (gpu-marked) the fused CUDA decoder."""
import os

import numpy as np
import pytest

import harness as H
import paper_1209_2137_b200 as P

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_vectors.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def arrays(gold):
    keys = sorted({k.rsplit("/", 1)[0] for k in gold if k.startswith("arr/")})
    for key in keys:
        name = key.split("/")[1]
        lens, nwords = gold[key + "/lens"], gold[key + "/nwords"]
        pay = np.split(gold[key + "/payload"], np.cumsum(nwords)[:-1])
        yield name, gold[key + "/values"], list(zip(lens.tolist(), pay))


def bad_chunks(gold, name):
    nw = gold[f"bad/{name}/nwords"]
    pays = np.split(gold[f"bad/{name}/payload"], np.cumsum(nw)[:-1])
    return pays, gold[f"bad/{name}/status"], gold[f"bad/{name}/decoded"]


def test_oracle_decodes_reference_vectors(oracle, gold):
    n = 0
    for name, vals, chunks in arrays(gold):
        st, out = oracle.decode_array(name, chunks)
        assert st == 0 and np.array_equal(out, vals), name
        n += 1
    assert n >= 12


def test_oracle_encodes_reference_vectors(oracle, gold):
    for name, vals, chunks in arrays(gold):
        mine = oracle.encode_array(name, vals)
        assert [c for c, _ in mine] == [c for c, _ in chunks]
        for (_, a), (_, b) in zip(mine, chunks):
            assert np.array_equal(a, b), name


def test_host_encoder_reproduces_reference_vectors(native, gold):
    for name, vals, chunks in arrays(gold):
        enc = H.encode_array(P.make_codec(name), vals)
        for i, (_, p) in enumerate(chunks):
            t = enc.table[i]
            assert np.array_equal(enc.words[int(t["word_off"]):][:int(t["n_words"])], p), name


def test_oracle_raw_widths(oracle, gold):
    for codec in ("simdbp128", "simdfastpfor"):
        for b in range(33):
            v = gold[f"raw/{codec}/{b}/values"]
            w = gold[f"raw/{codec}/{b}/payload"]
            st, out, used = oracle.decode_deltas(codec, w, len(v))
            assert st == 0 and used == len(w) and np.array_equal(out, v), (codec, b)


@pytest.mark.parametrize("name", ["simdbp128", "simdbp128-s4", "simdfastpfor", "simdfastpfor-s4"])
def test_oracle_statuses_on_reference_corruptions(oracle, gold, name):
    pays, stats, decs = bad_chunks(gold, name)
    for p, s, d in zip(pays, stats, decs):
        st, out = oracle.decode_chunk(name, p, 1500)
        assert st == s
        if s == 0:
            assert np.array_equal(out, d)


# ---- the fused CUDA decoder on the same vectors -------------------------

@pytest.mark.gpu
def test_gpu_decodes_reference_vectors(cuda, gold):
    for name, vals, chunks in arrays(gold):
        codec = P.make_codec(name)
        enc = P.layout(codec, [p for _, p in chunks], [c for c, _ in chunks])
        assert np.array_equal(P.decode_array(codec, enc), vals), name


@pytest.mark.gpu
def test_gpu_raw_widths(cuda, gold):
    for codec_name in ("simdbp128", "simdfastpfor"):
        codec = P.make_codec(codec_name)
        vals = [gold[f"raw/{codec_name}/{b}/values"] for b in range(33)]
        pays = [gold[f"raw/{codec_name}/{b}/payload"] for b in range(33)]
        enc = P.layout(codec, pays, [len(v) for v in vals])
        b = P.DeviceBatch(codec, enc, raw=True)
        b.decode()
        b.check()
        assert np.array_equal(b.output(), np.concatenate(vals))
        assert list(b.consumed[:33].cpu().numpy()) == [len(p) for p in pays]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["simdbp128", "simdbp128-s4", "simdfastpfor", "simdfastpfor-s4"])
def test_gpu_statuses_on_reference_corruptions(cuda, gold, name):
    pays, stats, decs = bad_chunks(gold, name)
    codec = P.make_codec(name)
    enc = P.layout(codec, pays, [1500] * len(pays))
    out, st = P.decode_array(codec, enc, return_status=True)
    assert list(st) == list(stats)
    for i, s in enumerate(stats):
        if s == 0:
            assert np.array_equal(out[1500 * i:1500 * (i + 1)], decs[i])
