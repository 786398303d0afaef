"""BASELINE.json config 4 (weighted MaxCut K32 / dense QUBO, n=32, p=8) on ONE B200:
E + full gradient without sharding (ket + bra + f64 table = 160 GiB of the 180 GB).
python tools/c4_single_gpu.py [qubo|wmaxcut]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n, p = 32, 8
os.environ["QAOA_MAX_QUBITS"] = str(n)
os.environ["QAOA_MEM_CEILING_BYTES"] = str(16 << n)
import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import rng


def qubo_polynomial(n: int, seed: int) -> qs.Polynomial:
    """Dense QUBO: n linear + n(n-1)/2 pair terms, weights (U-0.5)*8."""
    st = rng.Stream(seed)
    terms = [((st.next_uniform() - 0.5) * 8.0, 1 << i) for i in range(n)]
    for i in range(n):
        for j in range(i + 1, n):
            terms.append(((st.next_uniform() - 0.5) * 8.0, (1 << i) | (1 << j)))
    return qs.Polynomial(n, terms)


def weighted_maxcut(n: int, seed: int) -> qs.Polynomial:
    """Complete graph with integer weights 1 + floor(8U)."""
    st = rng.Stream(seed)
    edges = [(u, v, float(1 + int(8 * st.next_uniform()))) for u in range(n) for v in range(u + 1, n)]
    return qs.maxcut_polynomial(qs.Graph(n, edges))

kind = sys.argv[1] if len(sys.argv) > 1 else "qubo"
poly = qubo_polynomial(n, 1) if kind == "qubo" else weighted_maxcut(n, 1)
t0 = time.perf_counter()
h = qs.create_handle(poly, backend_name="b200")
h.ctx.synchronize()
t1 = time.perf_counter()
params = qs.linear_ramp_params(p)
qs.value_and_grad(h, params)
h.ctx.synchronize()
t2 = time.perf_counter()
v, g = qs.value_and_grad(h, params)
t3 = time.perf_counter()
print(f"C4 {kind} n={n} p={p} ({poly.num_terms} terms) on one B200: create_handle {t1 - t0:.2f} s, "
      f"E+grad {t3 - t2:.3f} s, E={v:.10f} in [{h.table.min_value}, {h.table.max_value}], "
      f"|grad|max={max(abs(x) for x in g.d_betas + g.d_gammas):.6f}")
