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
    from oracle.pyoracle import Oracle

    O = Oracle()
    wl = (48, "cluster", (20, 29), 0, bench.CODECS, "test")
    lo, hi = bench.plan_shards(wl, world)[rank]
    encs, expect, _ = bench.build_inputs(wl, lo, hi, threads=2)
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


def test_byte_balanced_shards_c5():
    """C5's per-array d varies (20..29): shards are contiguous and balanced
    by the bytes each array moves, not by array count."""
    import bench
    import harness as H

    wl = bench.WORKLOADS["c5"]
    d = H.array_widths(wl[0], wl[2], bench.SEED)
    w = bench.est_bytes_per_array(d, 2)
    for world in (1, 2, 4, 8):
        spans = bench.plan_shards(wl, world)
        assert spans[0][0] == 0 and spans[-1][1] == wl[0]
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        loads = [w[a:b].sum() for a, b in spans]
        assert max(loads) / min(loads) < 1 + 1e-3


def _run_bench(*argv, timeout=600):
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "MASTER_ADDR",
                        "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *argv], env=env,
                       capture_output=True, text=True, timeout=timeout, cwd=root)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return r.returncode, [json.loads(ln) for ln in lines], r.stderr


@pytest.mark.timeout(600)
def test_bench_spawns_ranks_for_gpus_n():
    """`bench.py --gpus 2` without a launcher spawns two ranks (here in the
    GPU-free --dry-run mode over gloo) and reports n_gpus == 2 with the
    workload split across both; --gpus 1 stays a single process."""
    rc, lines, err = _run_bench("--gpus", "2", "--dry-run", "--arrays", "40", "--steps", "1")
    assert rc == 0, err
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2
    spans = lines[0]["config"]["shards"]
    assert spans[0][0] == 0 and spans[1][1] == 40 and spans[0][1] == spans[1][0]
    assert all(n > 0 for n in lines[0]["config"]["arrays_per_rank"])
    rc, lines, err = _run_bench("--gpus", "1", "--dry-run", "--arrays", "8", "--steps", "1")
    assert rc == 0, err
    assert lines[0]["n_gpus"] == 1 and lines[0]["config"]["shards"] == [[0, 8]]


def test_bench_refuses_more_gpus_than_visible():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    rc, lines, _ = _run_bench("--gpus", "2", "--steps", "1", timeout=120)
    assert rc != 0 and "error" in lines[0]


@pytest.mark.timeout(600)
def test_reference_arm_loads_no_repo_library():
    """`bench.py --impl reference` runs the reference (oracle/_ref) alone: it
    imports neither the product package nor the harness and maps no repo
    shared library besides oracle/_ref, and reports the GPU arm's config
    keys on the full (here reduced) workload."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import runpy, sys, json\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--arrays', '64', '--steps', '1',"
        " '--warmup', '3']\n"
        "try:\n"
        "    runpy.run_path('bench.py', run_name='__main__')\n"
        "finally:\n"
        "    maps = [l.split()[-1] for l in open('/proc/self/maps') if l.rstrip().endswith('.so')]\n"
        "    mods = [m for m in sys.modules if m.split('.')[0] in ('paper_1209_2137_b200', 'harness')]\n"
        "    print('CHECK ' + json.dumps({'maps': sorted(set(maps)), 'mods': mods}))\n")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK")}
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    check = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("CHECK ")][0][6:])
    assert check["mods"] == []
    repo_libs = [m for m in check["maps"] if m.startswith(root)]
    assert repo_libs and all("/oracle/_ref/" in m for m in repo_libs), repo_libs
    assert line["impl"] == "reference" and line["config"]["verified"] is True
    assert line["config"]["arrays"] == 64 and line["config"]["codecs"] == ["simdbp128-s4",
                                                                         "simdfastpfor-s4"]
    assert line["cpu_baseline"]["cpu_model"]
