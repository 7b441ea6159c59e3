"""Per-SASS-instruction execution counts from an ncu report (SourceCounters):
totals per opcode and the hottest straight-line regions, per kernel.

    python tools/sass_hot.py REPORT.ncu-rep [--units N] [--top K] [--dump FILE]

--units: divide counts by N (e.g. warp iterations of 512 integers) so the
table reads as instructions per unit.
"""
import argparse
import collections
import csv
import io
import re
import subprocess

NCU = "/usr/local/cuda/bin/ncu"


def load(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    kernels, cur, rows = [], None, []
    for line in out.splitlines():
        if line.startswith('"Kernel Name"'):
            if cur:
                kernels.append((cur, rows))
            cur, rows = next(csv.reader(io.StringIO(line)))[1], []
            continue
        if line.startswith('"Address"'):
            header = next(csv.reader(io.StringIO(line)))
            continue
        r = next(csv.reader(io.StringIO(line)))
        if len(r) < 6:
            continue
        d = dict(zip(header, r))
        try:
            n = int(d["Instructions Executed"])
        except ValueError:
            continue
        samples = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        rows.append((d["Address"], d["Source"].strip(), n, samples))
    if cur:
        kernels.append((cur, rows))
    return kernels


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--units", type=float, default=1.0)
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--dump")
    a = ap.parse_args()
    seen = set()
    for name, rows in load(a.rep):
        tot = sum(n for _, _, n, _ in rows)
        if (name, tot) in seen:  # ncu lists some kernels twice
            continue
        seen.add((name, tot))
        print(f"== {name[:150]}\n   instructions executed {tot:,} ({tot / a.units:.1f} per unit)")
        ops = collections.Counter()
        for _, src, n, _ in rows:
            m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", src)
            ops[m.group(2) if m else src] += n
        for op, n in ops.most_common(a.top):
            print(f"   {op:12s} {n / a.units:8.1f}  {100 * n / tot:5.1f}%")
        if a.dump:
            with open(a.dump, "a") as f:
                f.write(f"== {name}\n")
                for addr, src, n, s in rows:
                    f.write(f"{n / a.units:9.2f} {s:6d}  {src}\n")


if __name__ == "__main__":
    main()
