#!/usr/bin/env python3
"""Benchmark: fused SIMD-BP128+D4 and SIMD-FastPFOR+D4 decode on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c5|c1|c4]

Workload (default c5 = BASELINE.json configs[4], the config the metric is
quoted on at 1/2/4/8 GPUs): 65,536 arrays x 65,536 sorted distinct uint32 from
the seeded BASELINE ClusterData recipe, d ~ U{20..29} per array, encoded with
simdbp128-s4 AND simdfastpfor-s4; arrays are partitioned by contiguous range
across the N ranks (strong scaling, no data-path collective).  One step decodes
the rank's shard under both codecs: one launch of the fused SIMD-BP128 kernel,
then izg_decode_ws's two SIMD-FastPFOR launches (page index pass + decode).

Timing: W warm-up steps, then K steps bracketed by a barrier and a device
synchronize, measured with CUDA events on the launching stream; the max over
ranks is reported (NCCL max-reduce).  Inputs (~8 GB) and outputs (16 GiB) per
step dwarf the 126 MB L2, so no flush is needed.  After timing, every rank
checksums its decoded output on the device and the mismatch count is
sum-reduced over NCCL (the only collective).

`e2e` repeats the metric through the host-buffer C ABI (izg_decode_host):
pinned host words in, decoded integers back to pinned host memory, all copies
inside the timed region.  `cpu_baseline` (rank 0, N=1) and `--impl reference`
time the reference library itself (compiled from its sources into
oracle/_ref) decoding a bounded sample of the same workload with every host
thread.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "G uint32/s decoded (BP128+D4, FastPFOR+D4) at 1/2/4/8 GPU; % of HBM roofline"
UNIT = "G uint32/s"
CODECS = ("simdbp128-s4", "simdfastpfor-s4")
N_INTS = 65536

WORKLOADS = {
    # name: (arrays, model, d (lo, hi), rate_ppm, codecs, description)
    "c5": (65536, "cluster", (20, 29), 0, CODECS,
           "C5 sharded whole-box decode: 65536 arrays x 65536 sorted ClusterData uint32 "
           "(BASELINE recipe, d~U{20..29} per array), simdbp128-s4 + simdfastpfor-s4"),
    "c1": (1024, "cluster", (29, 29), 0, ("simdbp128-s4",),
           "C1: 1024 arrays x 65536 ClusterData [0,2^29), simdbp128-s4"),
    "c4": (2048, "geometric", (32, 32), 100000, ("simdfastpfor-s4",),
           "C4: 2048 arrays x 65536, geometric(mean 8) gaps + 10% outliers U[2^12,2^24), "
           "simdfastpfor-s4 (prefix sums wrap mod 2^32)"),
}
SEED = 20120910


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def shard(n_arrays, world, rank):
    lo = n_arrays * rank // world
    hi = n_arrays * (rank + 1) // world
    return lo, hi


def build_inputs(P, wl, lo, hi, threads, want_values=False):
    """Generate arrays [lo, hi) in batches, encode with every codec, return
    per-codec Encoded (global out_off) plus the expected checksum."""
    n_arrays, model, d, rate, codecs, _ = wl
    batch = 2048
    enc_parts = {c: [] for c in codecs}
    word_base = {c: 0 for c in codecs}
    ck = np.zeros(2, dtype=np.uint64)
    sums = [0, 0]
    values_keep = []
    lib = P._native.lib()
    for b0 in range(lo, hi, batch):
        b1 = min(hi, b0 + batch)
        cnt = b1 - b0
        vals, _ = P.gen_arrays(model, cnt, N_INTS, d, seed=SEED + b0, rate_ppm=rate,
                               threads=threads)
        flat = vals.reshape(-1)
        lib.izg_checksum_host(P._native.ptr(flat), flat.size, (b0 - lo) * N_INTS, threads,
                              P._native.ptr(ck))
        sums[0] = (sums[0] + int(ck[0])) % (1 << 64)
        sums[1] ^= int(ck[1])
        offs = np.arange(cnt, dtype=np.uint64) * N_INTS
        counts = np.full(cnt, N_INTS, dtype=np.uint32)
        for c in codecs:
            e = P.encode_chunks(P.make_codec(c), flat, offs, counts,
                                allow_wrap=(model == "geometric"), threads=threads)
            e.table["word_off"] += np.uint64(word_base[c])
            e.table["out_off"] += np.uint64((b0 - lo) * N_INTS)
            word_base[c] += len(e.words)
            enc_parts[c].append(e)
        if want_values:
            values_keep.append(vals)
        del vals, flat
    encs = {}
    for c in codecs:
        words = np.concatenate([e.words for e in enc_parts[c]])
        table = np.concatenate([e.table for e in enc_parts[c]])
        encs[c] = P.Encoded(words, table)
    return encs, (sums[0], sums[1]), values_keep


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    PERIOD_MS = 20

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.PERIOD_MS)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def mark(self, start: bool):
        if start:
            self.t0 = time.perf_counter()
        else:
            self.t1 = time.perf_counter()

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t0", 0.0), getattr(self, "t1", float("inf"))
        # keep samples taken inside the timed region (nvidia-smi reports the
        # previous period, so allow one period of slack at the end)
        window = [ln for ts, ln in self.lines if t0 <= ts <= t1 + self.PERIOD_MS / 1e3]
        if not window and self.lines:
            window = [min(self.lines, key=lambda x: abs(x[0] - t0))[1]]
        for ln in window:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_sample(wl, threads, budget_s=12.0, sample_arrays=None):
    """The reference library (oracle/_ref, compiled from the reference's own
    sources) decoding a bounded sample of the workload with `threads` host
    threads: decode_array per array into pre-faulted per-array outputs."""
    import paper_1209_2137_b200 as P
    from oracle.pyoracle import Reference

    ref = Reference()
    n_arrays, model, d, rate, codecs, _ = wl
    m = sample_arrays or min(n_arrays, 1024)
    vals, _ = P.gen_arrays(model, m, N_INTS, d, seed=SEED, rate_ppm=rate, threads=threads)
    flat = vals.reshape(-1)
    offs = np.arange(m, dtype=np.uint64) * N_INTS
    counts = np.full(m, N_INTS, dtype=np.uint32)
    batches = []
    for c in codecs:
        # encoded by the reference itself (encode_array; the wrapping variant
        # for the C4 sums that exceed 2^32)
        if model == "geometric":
            payloads = [ref.encode_chunk_wrapping(c, vals[i]) for i in range(m)]
        else:
            payloads = [ref.encode_array(c, vals[i])[0][1] for i in range(m)]
        e = P.layout(P.make_codec(c), payloads, counts)
        b = ref.batch(c, e.words, e.table)
        b.decode(threads=threads)  # warm-up + correctness
        for i in (0, m - 1):
            if not np.array_equal(b.output(i, N_INTS), vals[i]):
                raise RuntimeError(f"reference decode mismatch on {c}")
        batches.append(b)
    return batches, m


def run_reference_arm(args, wl, world, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    batches, m = cpu_reference_sample(wl, threads)
    ints = m * N_INTS * len(batches)
    for _ in range(args.warmup):
        for b in batches:
            b.decode(threads=threads)
    times = []
    for _ in range(args.steps):
        t = sum(b.decode(threads=threads) for b in batches)
        times.append(t)
    tot = sum(times)
    value = ints * args.steps / tot / 1e9
    sample = (f"{m} of {wl[0]} arrays x {N_INTS} ints, {'+'.join(wl[4])}, one decode_array per "
              f"array per step, {threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * tot / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded BASELINE.json recipes; no dataset)",
        "config": {"workload": wl[5], "sample": sample},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = WORKLOADS[args.workload]
    world, rank, local = dist_init()

    if args.impl == "reference":
        run_reference_arm(args, wl, world, rank)
        return

    import torch

    import paper_1209_2137_b200 as P

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    threads = max(1, (os.cpu_count() or 1) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE",
                                                                          world))))
    n_arrays = wl[0]
    lo, hi = shard(n_arrays, world, rank)
    t0 = time.time()
    encs, expect, _ = build_inputs(P, wl, lo, hi, threads)
    prep_s = time.time() - t0

    # one output buffer shared by the codecs (each step rewrites it)
    out = torch.empty(max(e.n_out for e in encs.values()), dtype=torch.int32, device=dev)
    batches = {c: P.DeviceBatch(P.make_codec(c), encs[c], dev, out=out) for c in wl[4]}
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def step(events=None):
        for i, (c, b) in enumerate(batches.items()):
            if events is not None:
                events[c][0].record(stream)
            b.decode(stream)
            if events is not None:
                events[c][1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    for b in batches.values():
        b.check()

    kev = {c: [] for c in batches}
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize(dev)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.mark(True)
    start.record(stream)
    for _ in range(args.steps):
        ev = {c: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for c in batches}
        step(ev)
        for c in batches:
            kev[c].append(ev[c])
    end.record(stream)
    torch.cuda.synchronize(dev)
    clocks.mark(False)
    barrier()
    clk = clocks.stop()
    elapsed = start.elapsed_time(end) / 1e3
    kern_ms = {c: float(np.mean([a.elapsed_time(b) for a, b in kev[c]])) for c in batches}

    # correctness: device checksum of each codec's output vs the generated input
    mism = 0
    for c, b in batches.items():
        b.decode(stream)
        torch.cuda.synchronize(dev)
        b.check()
        if b.checksum() != expect:
            mism += 1
    t_el = torch.tensor([elapsed, float(mism)], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist

        mx = t_el[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t_el[1:].clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        elapsed, mism = float(mx.item()), int(sm.item())

    total_ints = n_arrays * N_INTS * len(batches)  # whole job, all ranks
    value = total_ints * args.steps / elapsed / 1e9

    # roofline of the dominant kernel (largest share of the step)
    peak, peak_kind = peaks()
    dom = max(kern_ms, key=kern_ms.get)
    alg_bytes = batches[dom].algorithmic_bytes
    achieved = alg_bytes / (kern_ms[dom] / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(args.workload, {}).get(dom)
            traffic = tr
    except Exception:
        pass

    # e2e through the host-buffer C ABI, pinned host memory, copies inside
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else min(args.steps, 3)
    h_words = {}
    h_tables = {}
    h2d = d2h = 0
    for c, e in encs.items():
        hw = torch.empty(len(e.words), dtype=torch.int32, pin_memory=True)
        hw.numpy().view(np.uint32)[:] = e.words
        h_words[c] = hw
        h_tables[c] = e.table
        h2d += e.words.nbytes + e.table.nbytes
        d2h += 4 * e.n_out + 4 * len(e.table)
    n_out = max(e.n_out for e in encs.values())
    h_out = torch.empty(n_out, dtype=torch.int32, pin_memory=True)
    h_status = np.zeros(max(len(e.table) for e in encs.values()), dtype=np.int32)
    lib = P._native.lib()

    def e2e_step():
        for c in batches:
            codec = P.make_codec(c)
            rc = lib.izg_decode_host(codec.codec, codec.delta, h_words[c].data_ptr(),
                                     len(encs[c].words), P._native.ptr(h_tables[c]),
                                     len(h_tables[c]), h_out.data_ptr(), n_out,
                                     P._native.ptr(h_status))
            if rc != 0:
                raise RuntimeError(f"izg_decode_host failed: {rc}")

    e2e_step()  # warm-up (scratch allocation)
    barrier()
    te = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    te = time.perf_counter() - te
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([te], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        te = float(t.item())
    e2e_value = total_ints * e2e_steps / te / 1e9
    # last e2e step's output must equal the last codec's decode
    last = list(batches)[-1]
    ck = np.zeros(2, dtype=np.uint64)
    lib.izg_checksum_host(h_out.data_ptr(), encs[last].n_out, 0, threads, P._native.ptr(ck))
    e2e_ok = (int(ck[0]), int(ck[1])) == expect

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cthreads = os.cpu_count() or 1
            cb, m = cpu_reference_sample(wl, cthreads)
            tt, reps, t_start = 0.0, 0, time.time()
            while time.time() - t_start < 12.0 and reps < 200:
                tt += sum(b.decode(threads=cthreads) for b in cb)
                reps += 1
            cval = m * N_INTS * len(cb) * reps / tt / 1e9
            cpu = {"value": round(cval, 4), "unit": UNIT, "cores": cthreads, "kind": "reference",
                   "sample": f"{m} arrays x {N_INTS} ints of this workload, {'+'.join(wl[4])}, "
                             f"{reps} passes of decode_array per array on {cthreads} threads "
                             f"(reference compiled from source, oracle/_ref)"}
        except Exception as ex:  # reference library absent on this box
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank == 0:
        bits = {c: round(32 * encs[c].payload_words / ((hi - lo) * N_INTS), 3) for c in encs}
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * elapsed / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (seeded BASELINE.json recipes; no dataset)",
            "config": {
                "workload": wl[5], "arrays": n_arrays, "ints_per_array": N_INTS,
                "codecs": list(batches), "bits_per_int_rank0": bits,
                "ms_per_launch_rank0": {c: round(v, 4) for c, v in kern_ms.items()},
                "l2": "inputs+outputs per step >> 126 MB L2 (no flush needed)",
                "parallelism": f"shard by array over {world} rank(s); NCCL only for the "
                               "final checksum and timing reduction",
                "verified": mism == 0, "prep_s_rank0": round(prep_s, 1),
            },
            "roofline": {"bound": "hbm",
                         "kernel": (f"fp_index_kernel+decode_kernel[{dom}] (events around both)"
                                    if batches[dom].launches_per_decode == 2
                                    else f"decode_kernel[{dom}]"),
                         "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "peak_source": peak_kind,
                         "traffic": traffic,
                         "algorithmic_bytes_per_launch": alg_bytes},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    "path": "izg_decode_host (pinned host buffers; H2D + decode on 4 slot streams, D2H split over 3 streams)",
                    "verified": e2e_ok},
            "clocks": clk,
            "gpu_launches": args.steps * sum(b.launches_per_decode for b in batches.values()),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    if mism:
        sys.exit(1)


if __name__ == "__main__":
    main()
