"""Summarise `ncu --set full` reports for profiles/: per kernel launch, the
HBM traffic and throughput, shared-memory bank conflicts, issue activity,
occupancy and the top warp stall reasons (north_star: "each kernel choice
is evidenced by ncu counters").

    python tools/ncu_summary.py gpurun_out/prof_c5.ncu-rep [...] > profiles/rXX_ncu_<cfg>.txt

Reads `ncu -i <rep> --page raw --csv` (ncu is in this container; no GPU
needed to read a report).
"""
import csv
import io
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem ld wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "smem st wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st bank conflicts"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]
STALL_PREFIX = "smsp__average_warps_issue_stalled_"
STALL_SUFFIX = "_per_issue_active.ratio"


def rows_of(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rd = list(csv.reader(io.StringIO(out)))
    hdr, units = rd[0], rd[1]
    return hdr, units, rd[2:]


def fmt(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    if unit in ("byte", "Kbyte", "Mbyte", "Gbyte"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
        return f"{x * scale / 1e9:.3f} GB"
    if unit in ("nsecond", "usecond", "msecond"):
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}[unit]
        return f"{x * scale:.3f} ms"
    return f"{x:,.2f} {unit}".strip()


def main(reps):
    for rep in reps:
        hdr, units, rows = rows_of(rep)
        col = {h: i for i, h in enumerate(hdr)}
        for r in rows:
            name = r[col["Kernel Name"]]
            print(f"== {rep}: {name[:110]}")
            for key, label in KEYS:
                if key in col:
                    print(f"  {label:26s} {fmt(r[col[key]], units[col[key]])}")
            stalls = []
            for h, i in col.items():
                if h.startswith(STALL_PREFIX) and h.endswith(STALL_SUFFIX) and "selected" not in h:
                    try:
                        stalls.append((float(r[i].replace(",", "")), h[len(STALL_PREFIX):-len(STALL_SUFFIX)]))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            tot = sum(s for s, _ in stalls) or 1.0
            print("  top warp stall reasons (warps stalled per issue-active cycle, share):")
            for s, n in stalls[:6]:
                print(f"    {n:24s} {s:7.2f}  {100 * s / tot:5.1f}%")
            print()


if __name__ == "__main__":
    main(sys.argv[1:])
