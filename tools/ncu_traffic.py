"""Summarise an `ncu --set full` capture of k_sweep launches per sweep kind.

    python tools/ncu_traffic.py REPORT.ncu-rep [--json profiles/traffic.json] [--alg N]

Each launch's template arguments (shape, NV, ..., MODE, ...) name its kind the same
way the live profiler does (DeviceContext.prof_kind_name): 'single_B',
'braket_merged_A', ...  For every kind: launches, mean duration, DRAM bytes read +
written per launch (the `traffic` field bench.py reports), achieved DRAM GB/s, FP64 /
shared-memory pipe utilisation and the top stall reasons.  --json writes
{kind: bytes_per_launch} for bench.py.
"""

from __future__ import annotations

import argparse
import csv
import json
import re
import subprocess
from collections import defaultdict

A_SHAPES = {0, 1, 3, 4, 6}  # SH_A1, SH_A1X, SH_A2, SH_A2X, SH_A3 (sweep.cuh)


def kind_of(name: str) -> str | None:
    m = re.search(r"k_sweep<([^>]*)>", name)
    if not m:
        return None
    args = [int(x) for x in re.findall(r"(\d+)", re.sub(r"\(\w+(?: \w+)?\)", "", m.group(1)))]
    if len(args) < 6:
        return None
    sh, nv, mode = args[0], args[1], args[5]
    return f"{'single' if nv == 1 else 'braket'}{['', '_merged', '_bridge'][mode]}_{'A' if sh in A_SHAPES else 'B'}"


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--json")
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[0]

    units = rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}

    def col(r, name, default=0.0):
        try:
            i = hdr.index(name)
            return float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
        except (ValueError, IndexError):
            return default

    stall_cols = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
    agg = defaultdict(lambda: defaultdict(float))
    for r in rows[2:]:
        k = kind_of(r[hdr.index("Kernel Name")])
        if k is None:
            continue
        a = agg[k]
        a["launches"] += 1
        a["ms"] += col(r, "gpu__time_duration.sum")
        a["rd"] += col(r, "dram__bytes_read.sum")
        a["wr"] += col(r, "dram__bytes_write.sum")
        a["fp64"] += col(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
        a["smem"] += col(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")
        a["issue"] += col(r, "smsp__issue_active.avg.pct_of_peak_sustained_active")
        a["regs"] = col(r, "launch__registers_per_thread")
        for h in stall_cols:
            a["stall:" + h.replace("smsp__pcsamp_warps_issue_stalled_", "")] += col(r, h)
    out = {}
    for k in sorted(agg):
        a = agg[k]
        n = a["launches"]
        byt = (a["rd"] + a["wr"]) / n
        out[k] = byt
        ms = a["ms"] / n
        st = sorted(((v, h[6:]) for h, v in a.items() if h.startswith("stall:")), reverse=True)
        tot = sum(v for v, _ in st) or 1.0
        top = ", ".join(f"{h} {100 * v / tot:.0f}%" for v, h in st[:4])
        print(f"{k:18s} x{int(n)} {ms:7.2f} ms  dram rd {a['rd'] / n / 1e9:6.2f} + wr {a['wr'] / n / 1e9:6.2f} GB "
              f"= {byt / (ms * 1e-3) / 1e9:6.0f} GB/s  fp64 {a['fp64'] / n:4.1f}%  smem {a['smem'] / n:4.1f}%  "
              f"issue {a['issue'] / n:4.1f}%  regs {int(a['regs'])} | {top}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump({k: round(v) for k, v in out.items()}, f, indent=1)


if __name__ == "__main__":
    main()
