"""Z2-reduced vs full fast path on small cases: max |diff| of statevectors and <C>."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2407_13012_b200 as qs
from oracle import oracle

n = int(sys.argv[1]) if len(sys.argv) > 1 else 21
poly = qs.maxcut_polynomial(qs.random_regular(n, 3, seed=1) if n % 2 == 0 else qs.erdos_renyi(n, 0.3, seed=1))
table = oracle.precompute_table(poly.weights, poly.masks, n)
h = qs.create_handle(poly, backend_name="b200")
for betas, gammas in (([0.0], [0.0]), ([0.0], [0.7]), ([0.3], [0.0]), ([0.3], [0.7]), ([0.3, 0.2], [0.7, -0.4]),
                      ([0.3, 0.2, 0.5], [0.7, -0.4, 0.2])):
    prm = qs.QaoaParams(betas, gammas)
    want = oracle.simulate(table, n, prm.gammas, prm.betas)
    os.environ["QSB_NO_SYM"] = "0"
    got = qs.statevector(h, prm)
    e = qs.expectation(h, prm)
    v, g = qs.value_and_grad(h, prm)
    os.environ["QSB_NO_SYM"] = "1"
    v1, g1 = qs.value_and_grad(h, prm)
    d = np.abs(got - want)
    lo = d[: 1 << (n - 1)].max(); hi = d[1 << (n - 1):].max()
    print(f"p={prm.p} b={betas} g={gammas}: |psi-oracle| lower {lo:.2e} upper {hi:.2e}; E {e:.12f} vs "
          f"{oracle.expectation(table, want):.12f}; vg {v:.12f} vs nosym {v1:.12f}; "
          f"grad diff {np.max(np.abs(np.array(g.d_betas + g.d_gammas) - np.array(g1.d_betas + g1.d_gammas))):.2e}")
