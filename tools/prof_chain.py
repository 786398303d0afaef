"""One value_and_grad of MaxCut reg3 n (default 28), depth p (default 3) through the
public API -- the target of focused ncu captures of single window-chain sweeps:

    ncu --set full --import-source on --clock-control none -k regex:k_sweep \\
        --launch-skip 8 --launch-count 1 -o gpurun_out/merged_A python tools/prof_chain.py 28 3

At p=3 the chain's 13 sweeps are: A | B1 | B2B2 | B1 | AA (single merged A) | B1 |
B2B2 (bridge) | B1 | AA (bra/ket merged A) | B1 | B2B2 (bra/ket merged B) | B1 | A."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_13012_b200 as qs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
p = int(sys.argv[2]) if len(sys.argv) > 2 else 3
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
os.environ.setdefault("QAOA_MAX_QUBITS", str(max(30, n)))
os.environ.setdefault("QAOA_MEM_CEILING_BYTES", str(max(16 << 30, 16 << n)))
h = qs.create_handle(qs.maxcut_polynomial(qs.random_regular(n, 3, seed=1)), backend_name="b200")
for _ in range(reps):
    v, g = qs.value_and_grad(h, qs.linear_ramp_params(p))
h.ctx.synchronize()
print(f"n={n} p={p} E={v!r}")
