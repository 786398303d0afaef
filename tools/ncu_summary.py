"""Summarise an ncu report: per-kernel duration, DRAM, issue and top stall reasons."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]


def col(r, name):
    return r[hdr.index(name)] if name in hdr else ""


stalls = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
for r in rows[2:]:
    name = col(r, "Kernel Name")
    dur = float(col(r, "gpu__time_duration.sum") or 0)
    rd = float(col(r, "dram__bytes_read.sum") or 0)
    wr = float(col(r, "dram__bytes_write.sum") or 0)
    pct = col(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
    regs = col(r, "launch__registers_per_thread")
    ipc = col(r, "smsp__issue_active.avg.pct_of_peak_sustained_active")
    inst = float(col(r, "smsp__inst_executed.sum") or 0)
    st = sorted(((float(col(r, h) or 0), h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h in stalls), reverse=True)
    tot = sum(v for v, _ in st) or 1
    top = ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in st[:6])
    print(f"{name[:34]:34s} {dur:7.2f}ms dram {pct:>6s}% rd {rd:5.2f} wr {wr:5.2f} GB regs {regs} issue {ipc}% inst {inst/1e6:.0f}M | {top}")
