"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) per kernel.

    python tools/ncu_launches.py LAUNCHES.csv HEADER_LINE... > profiles/<round>_launches.txt
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
tot = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    ms = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    name = r[ik].split("(")[0] if "(" in r[ik] else r[ik]
    tot[name][0] += 1
    tot[name][1] += ms
total = sum(v[1] for v in tot.values())
for line in sys.argv[2:]:
    print("# " + line)
print(f"# total {total:.1f} ms over {sum(v[0] for v in tot.values())} launches")
for k, (n, ms) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{ms:9.2f} ms {100 * ms / total:5.1f}% {n:4d}x  {k}")
