#!/bin/bash
# A/B of sweep-family env knobs on the C3 bench (5 steps each, interleaved twice):
#   tools/ab_families.sh "" "QSB_SWEEP_R1MB=6" "QSB_SWEEP_R1MB=4" ...
for rep in 1 2; do
  for cfg in "$@"; do
    out=$(env $cfg python bench.py --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1)
    python - "$cfg" "$out" <<'PY'
import json, sys
d = json.loads(sys.argv[2])
k = d["kernels"]
# the expectation is printed so a variant that computes something else shows up at once
print(f"[{sys.argv[1] or 'default'}] {d['ms_per_step']:.1f} ms  E={d['expectation']:.12f}  " +
      " ".join(f"{n}={v['ms_per_step']:.1f}" for n, v in sorted(k.items())))
PY
  done
done
