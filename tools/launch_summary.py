"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch
list of `bench.py` (C5): per decode-path kernel, launches, mean duration and
share of the device-resident decode step.  Launches of the e2e pieces are
excluded by size (the step's launches are the long ones).

    python tools/launch_summary.py gpurun_out/final/launches_c5.csv
"""
import csv
import collections
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
dur = collections.defaultdict(list)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum" or "izg::" not in r[ki] or "checksum" in r[ki]:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    v = float(r[vi].replace(",", ""))
    unit = r[h.index("Metric Unit")]
    us = v / 1e3 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1e3
    dur[name].append(us)
# the step's launches are the long ones (>= 0.3 ms at C5; the lane index pass takes 0.5 ms)
step = {k: [x for x in v if x >= 300.0] for k, v in dur.items()}
tot = sum(sum(v) / len(v) for v in step.values() if v)
for k, v in step.items():
    if v:
        m = sum(v) / len(v)
        print(f"{k:40s} launches={len(v)}  mean={m:9.1f} us  share_of_step={100 * m / tot:5.1f}%")
