#!/bin/bash
# print per-kind sweep times from a bench.py JSON log: tools/bench_kinds.sh LOG...
for f in "$@"; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "ms/step", round(d["ms_per_step"], 1), "simulate", round(d["simulate_ms"], 1))
for k, v in d["kernels"].items():
    print(f"    {k:18s} {v['ms_per_step']:7.2f} ms  x{v['launches_per_step']:.0f}  {v['frac']:.3f}")
PY
done
