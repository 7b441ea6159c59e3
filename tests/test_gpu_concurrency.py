"""Concurrent use of the C ABI (the reference is reentrant on disjoint buffers,
SPEC.md:208-209): several host threads in izg_decode_host at once (per-thread
scratch, shared device state), and device decodes racing on separate streams
(per-launch claim counters)."""
import threading

import numpy as np
import pytest
import torch

import harness as H
import paper_1209_2137_b200 as P

pytestmark = pytest.mark.gpu


def arrays(seed, k=6):
    vals, _ = H.gen_arrays("cluster", k, 65536, 26, seed=seed)
    return vals.reshape(-1)


def test_host_threads(cuda):
    names = ["simdbp128-s4", "simdfastpfor-s4", "bp32", "simplepfor-s4"]
    work = []
    for i, name in enumerate(names * 2):
        codec = P.make_codec(name)
        flat = arrays(100 + i)
        if codec.codec in (0, 1):
            enc = H.encode_array(codec, flat)
        else:
            from oracle.pyoracle import Reference

            ch = Reference().encode_array(name, flat)
            enc = P.layout(codec, [p for _, p in ch], [n for n, _ in ch])
        work.append((codec, enc, flat))
    errors = []

    def run(codec, enc, flat):
        try:
            for _ in range(3):
                got = P.decode_array(codec, enc)
                if not np.array_equal(got, flat):
                    errors.append(codec.name)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ts = [threading.Thread(target=run, args=w) for w in work]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_streams_race(cuda):
    codec = P.make_codec("simdfastpfor-s4")
    batches, flats = [], []
    for i in range(4):
        flat = arrays(200 + i, k=16)
        batches.append(P.DeviceBatch(codec, H.encode_array(codec, flat)))
        flats.append(flat)
    streams = [torch.cuda.Stream() for _ in batches]
    for _ in range(5):
        for b, s in zip(batches, streams):
            b.decode(s)
    torch.cuda.synchronize()
    for b, flat in zip(batches, flats):
        b.check()
        assert np.array_equal(b.output(), flat)
