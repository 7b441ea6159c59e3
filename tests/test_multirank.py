"""Multi-rank host logic on CPU (gloo, world_size 2): the bench's array
sharding covers the workload exactly once, every rank's shard decodes (here
with the oracle, as the GPU is absent) to its expected checksum, and the
timing/mismatch reductions behave as bench.py uses them."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_1209_2137_b200 as P
    from oracle.pyoracle import Oracle

    O = Oracle()
    wl = (48, "cluster", (20, 29), 0, bench.CODECS, "test")
    lo, hi = bench.shard(wl[0], world, rank)
    encs, expect, _ = bench.build_inputs(P, wl, lo, hi, threads=2)
    mism = 0
    for name, e in encs.items():
        out = np.zeros(e.n_out, np.uint32)
        for t in e.table:
            w = e.words[int(t["word_off"]):][:int(t["n_words"])]
            st, dec = O.decode_chunk(name, w, int(t["n"]))
            assert st == 0
            out[int(t["out_off"]):int(t["out_off"]) + int(t["n"])] = dec
        from paper_1209_2137_b200.device import host_checksum

        if host_checksum(out) != expect:
            mism += 1
    rng = torch.tensor([lo, hi], dtype=torch.int64)
    ranges = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(ranges, rng)
    m = torch.tensor([float(mism)])
    dist.all_reduce(m, op=dist.ReduceOp.SUM)
    t = torch.tensor([0.5 + rank])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        with open(os.path.join(result_dir, "r.txt"), "w") as f:
            f.write(f"{[tuple(r.tolist()) for r in ranges]}|{m.item()}|{t.item()}")
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharding_and_reductions(tmp_path, native, oracle):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    ranges, mism, tmax = open(tmp_path / "r.txt").read().split("|")
    ranges = eval(ranges)
    assert ranges[0][0] == 0 and ranges[-1][1] == 48
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    assert float(mism) == 0.0
    assert float(tmax) == 1.5


def test_shard_partition_all_world_sizes():
    import bench

    for world in (1, 2, 3, 4, 8):
        spans = [bench.shard(65536, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 65536
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
