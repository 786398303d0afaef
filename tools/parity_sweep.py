"""Extended parity sweep on the GPU box: random instances (MaxCut families, weighted
integer MaxCut, float QUBO), n = 12..26, p = 1..6, random angles, fast mode -- B200
value_and_grad / expectation / statevector vs the CPU oracle (the reference's numba
arithmetic).  Writes a table; every row must be within the north star's 1e-10.
python tools/parity_sweep.py OUT.txt [count]"""
import os, sys, time
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))
import numpy as np
import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import rng
from conftest import random_instance
from oracle import oracle


def qubo(n, seed):
    st = rng.Stream(seed)
    terms = [((st.next_uniform() - 0.5) * 8.0, 1 << i) for i in range(n)]
    terms += [((st.next_uniform() - 0.5) * 8.0, (1 << i) | (1 << j)) for i in range(n) for j in range(i + 1, n)
              if st.next_uniform() < 0.4]
    return qs.Polynomial(n, terms), "qubo"


def wmaxcut(n, seed):
    st = rng.Stream(seed)
    edges = [(u, v, float(1 + int(8 * st.next_uniform()))) for u in range(n) for v in range(u + 1, n)
             if st.next_uniform() < 0.5]
    return qs.maxcut_polynomial(qs.Graph(n, edges)), "wmaxcut"


out_path = sys.argv[1]
count = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rs = np.random.default_rng(2026)
rows, worst = [], 0.0
t_start = time.perf_counter()
for k in range(count):
    n = int(rs.integers(12, 27))
    p = int(rs.integers(1, 7))
    kind = k % 3
    if kind == 0:
        poly, fam = random_instance(7000 + k, n), "maxcut"
    elif kind == 1:
        poly, fam = wmaxcut(n, 8000 + k)
    else:
        poly, fam = qubo(n, 9000 + k)
    params = qs.QaoaParams(list(rs.uniform(-np.pi, np.pi, p)), list(rs.uniform(-2, 2, p)))
    h = qs.create_handle(poly, backend_name="b200")
    v, g = qs.value_and_grad(h, params)
    e = qs.expectation(h, params)
    psi = np.asarray(qs.statevector(h, params))
    table = np.asarray(h.table.values.data)
    qs.simulate(h, params)  # a Z2-reduced state (MaxCut) is drawn from its lower half
    ss = qs.draw(h, 2000, k)
    want_idx, want_cost = oracle.sample(np.asarray(h.state.data), table, 2000, k)
    d_ok = bool(np.array_equal(ss.indices, want_idx) and np.array_equal(ss.costs, want_cost))
    h.close()
    want_t = oracle.precompute_table(poly.weights, poly.masks, n)
    want_psi = oracle.simulate(want_t, n, params.gammas, params.betas)
    want_e = oracle.expectation(want_t, want_psi)
    dg, db = oracle.gradient(want_t, want_psi.copy(), params.gammas, params.betas)
    got = np.concatenate([np.array(g.d_gammas), np.array(g.d_betas)])
    want = np.concatenate([dg, db])
    e_err = max(abs(v - want_e), abs(e - want_e)) / max(1.0, abs(want_e))
    g_err = float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300))
    s_err = float(np.max(np.abs(psi - want_psi)) / np.max(np.abs(want_psi)))
    t_ok = bool(np.array_equal(table, want_t)) and d_ok
    worst = max(worst, e_err, g_err, s_err)
    rows.append(f"{k:3d} {fam:8s} n={n:2d} p={p} terms={poly.num_terms:4d}  table+draws bit-exact={t_ok}  "
                f"E rel {e_err:.2e}  grad rel {g_err:.2e}  psi rel {s_err:.2e}")
    print(rows[-1], flush=True)
with open(out_path, "w") as f:
    f.write(f"# tools/parity_sweep.py: {count} random instances, B200 fast mode vs the CPU oracle "
            f"(numba arithmetic), worst relative error {worst:.2e} (bar 1e-10); {time.perf_counter() - t_start:.0f} s\n")
    f.write("\n".join(rows) + "\n")
print("worst", worst)
