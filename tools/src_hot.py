"""Per-source-line executed instructions and stall samples from an ncu report
captured with --import-source on (ncu --page source --print-source sass,cuda).

    python tools/src_hot.py REPORT.ncu-rep [--units N] [--min X] [--kernel SUBSTR]
"""
import argparse, csv, io, subprocess, collections, os

ap = argparse.ArgumentParser()
ap.add_argument("rep"); ap.add_argument("--units", type=float, default=1.0)
ap.add_argument("--min", type=float, default=0.5); ap.add_argument("--kernel", default="")
a = ap.parse_args()
out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", a.rep, "--page", "source", "--csv",
                      "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
fpath, fn, hdr = None, None, None
rows = collections.OrderedDict()
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fpath = os.path.basename(r[1]); continue
    if r[0] == "Function Name": fn = r[1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < len(hdr) - 2 or not r[0].isdigit(): continue
    if a.kernel and a.kernel not in (fn or ""): continue
    d = dict(zip(hdr, r))
    try: n = int(d["Instructions Executed"]); s = int(d["Warp Stall Sampling (All Samples)"])
    except (ValueError, KeyError): continue
    key = (fpath, int(r[0]))
    if key in rows: rows[key][0] += n; rows[key][1] += s
    else: rows[key] = [n, s, r[1].strip()]
tot = sum(v[0] for v in rows.values()); ts = sum(v[1] for v in rows.values()) or 1
print(f"total {tot / a.units:.1f} per unit, {ts} samples")
byfile = collections.Counter()
for (f, l), (n, s, src) in rows.items(): byfile[f] += n
for f, n in byfile.most_common(): print(f"  {f:28s} {n / a.units:8.1f}")
for (f, l), (n, s, src) in sorted(rows.items()):
    if n / a.units >= a.min or 100 * s / ts >= 1.0:
        print(f"{f:22s}:{l:4d} {n / a.units:7.1f} {100 * s / ts:5.1f}%  {src[:90]}")
