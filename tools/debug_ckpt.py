"""value_and_grad with / without forward checkpoints and deferred scaling, several n, p."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2407_13012_b200 as qs
from oracle import oracle

for n in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["16", "22"])]:
    for p in (1, 2, 3):
        poly = qs.maxcut_polynomial(qs.random_regular(n, 3, seed=p) if n % 2 == 0 else qs.erdos_renyi(n, 0.4, seed=p))
        table = oracle.precompute_table(poly.weights, poly.masks, n)
        prm = qs.QaoaParams([0.3, -0.2, 0.5][:p], [0.7, -0.4, 0.2][:p])
        e, dg, db = oracle.value_and_grad(table, n, prm.gammas, prm.betas)
        h = qs.create_handle(poly, backend_name="b200")
        out = []
        for env in ({}, {"QSB_NO_CKPT": "1"}, {"QSB_NO_CKPT": "1", "QSB_NO_DEFER": "1"}, {"QSB_NO_SYM": "1"},
                    {"QSB_NO_SYM": "1", "QSB_NO_CKPT": "1"}):
            for k in ("QSB_NO_CKPT", "QSB_NO_DEFER", "QSB_NO_SYM"):
                os.environ.pop(k, None)
            os.environ.update(env)
            v, g = qs.value_and_grad(h, prm)
            err = np.max(np.abs(np.array(g.d_betas) - db)), np.max(np.abs(np.array(g.d_gammas) - dg))
            out.append(f"{env or 'default'}: db {err[0]:.1e} dg {err[1]:.1e}")
        print(f"n={n} p={p}: " + " | ".join(out))
        h.close()
