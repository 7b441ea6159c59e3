"""Print kernel / metric / value triples of an `ncu --csv --log-file` launch list."""
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    for r in rows[1:]:
        if "elementwise" in r[ki]:
            continue
        print(r[ki].split("(")[0][:44], r[mi], r[vi])
