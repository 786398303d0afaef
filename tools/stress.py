"""Race hunt: repeat value_and_grad / simulate / draw many times on several sizes and
require bit-identical results every time (any TMA-ring / barrier / cluster race shows
up as nondeterminism).  python tools/stress.py seconds"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2407_13012_b200 as qs
from conftest import random_instance

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
cases = []
for n in (13, 17, 21, 24, 27):
    poly = random_instance(1234 + n, n)
    h = qs.create_handle(poly, backend_name="b200")
    rs = np.random.default_rng(n)
    params = qs.QaoaParams(list(rs.uniform(-2, 2, 3)), list(rs.uniform(-1, 1, 3)))
    v, g = qs.value_and_grad(h, params)
    qs.simulate(h, params)
    ss = qs.draw(h, 50000, 9)
    psi = np.asarray(h.state.data).copy()
    cases.append((n, h, params, v, tuple(g.d_betas) + tuple(g.d_gammas), psi, ss.indices.copy()))
t0, it, bad = time.perf_counter(), 0, 0
while time.perf_counter() - t0 < budget:
    for n, h, params, v0, g0, psi0, idx0 in cases:
        v, g = qs.value_and_grad(h, params)
        if v != v0 or tuple(g.d_betas) + tuple(g.d_gammas) != g0:
            bad += 1
            print(f"MISMATCH value_and_grad n={n} iter {it}", flush=True)
        qs.simulate(h, params)
        if not np.array_equal(np.asarray(h.state.data), psi0):
            bad += 1
            print(f"MISMATCH statevector n={n} iter {it}", flush=True)
        if not np.array_equal(qs.draw(h, 50000, 9).indices, idx0):
            bad += 1
            print(f"MISMATCH draw n={n} iter {it}", flush=True)
    it += 1
print(f"stress: {it} rounds x {len(cases)} sizes in {time.perf_counter() - t0:.0f} s, mismatches: {bad}")
