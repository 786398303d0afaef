"""Per-source-line warp-stall breakdown of one kernel in an ncu report (needs
-lineinfo and --import-source on):  python tools/ncu_lines.py REPORT.ncu-rep [TOP]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, lines = None, None, []
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0].isdigit() and hdr and len(r) == len(hdr):
        lines.append((cur, int(r[0]), r[1], r))
reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


out = [(num(r[4]), f, ln, src.strip()[:84], [(h, num(r[i])) for i, h in reasons]) for f, ln, src, r in lines]
out = [o for o in out if o[0]]
tot = sum(o[0] for o in out)
agg = collections.Counter()
for o in out:
    for h, v in o[4]:
        agg[h] += v
print(f"samples {tot}: " + ", ".join(f"{h[6:]} {100 * v / tot:.1f}%" for h, v in agg.most_common(10)))
for s, f, ln, src, rs in sorted(out, reverse=True)[:top]:
    t3 = sorted(rs, key=lambda x: -x[1])[:3]
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<5d} {src:84s} | " + ", ".join(f"{h[6:]} {100 * v / tot:.1f}" for h, v in t3))
