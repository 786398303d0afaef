"""QSB_NO_DEFER=1 (every sweep stores true values) under the A/B knobs, n=16 p=2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2407_13012_b200 as qs
from oracle import oracle

n, p = int(sys.argv[1]) if len(sys.argv) > 1 else 16, 2
poly = qs.maxcut_polynomial(qs.random_regular(n, 3, seed=p))
table = oracle.precompute_table(poly.weights, poly.masks, n)
prm = qs.QaoaParams([float(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0.3", "-0.2"])], [0.7, -0.4])
e, dg, db = oracle.value_and_grad(table, n, prm.gammas, prm.betas)
h = qs.create_handle(poly, backend_name="b200")
base = {"QSB_NO_DEFER": "1", "QSB_NO_CKPT": "1", "QSB_NO_SYM": "1"}
for extra in ({}, {"QSB_STAG": "0"}, {"QSB_STAGP": "0"}, {"QSB_NO_MERGE": "1"}, {"QSB_STAG": "0", "QSB_STAGP": "0"},
              {"QSB_NO_MERGE": "1", "QSB_STAGP": "0"}, {"QSB_NO_DEFER": "0"}):
    env = dict(base, **extra)
    for k in ("QSB_NO_DEFER", "QSB_NO_CKPT", "QSB_NO_SYM", "QSB_STAG", "QSB_STAGP", "QSB_NO_MERGE", "QSB_DBG_NO_KEEP"):
        os.environ.pop(k, None)
    os.environ.update(env)
    v, g = qs.value_and_grad(h, prm)
    sv = qs.statevector(h, prm)
    psi = oracle.simulate(table, n, prm.gammas, prm.betas)
    print(extra, f"E {abs(v - e):.1e} db {np.max(np.abs(np.array(g.d_betas) - db)):.1e} "
          f"dg {np.max(np.abs(np.array(g.d_gammas) - dg)):.1e} psi {np.max(np.abs(sv - psi)):.1e}")
