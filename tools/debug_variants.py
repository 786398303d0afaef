"""value_and_grad vs the oracle under the sweep-family knobs (run with QSB_LIB=... to
pick the product or the variant library)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2407_13012_b200 as qs
from oracle import oracle

KNOBS = [{}, {"QSB_NO_CKPT": "1"}, {"QSB_STAGP": "0"}, {"QSB_STAGP": "0", "QSB_NO_CKPT": "1"}, {"QSB_STAG": "0"},
         {"QSB_STAG": "0", "QSB_NO_CKPT": "1"}, {"QSB_NO_MERGE": "1"}]
print("variants:", qs._lib.has_variants() if hasattr(qs._lib, "has_variants") else "?")
for n in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["13", "16", "21"])]:
    for p in (1, 3):
        poly = qs.maxcut_polynomial(qs.erdos_renyi(n, 0.4, seed=p))
        table = oracle.precompute_table(poly.weights, poly.masks, n)
        prm = qs.QaoaParams([0.3, -0.2, 0.5][:p], [0.7, -0.4, 0.2][:p])
        e, dg, db = oracle.value_and_grad(table, n, prm.gammas, prm.betas)
        h = qs.create_handle(poly, backend_name="b200")
        out = []
        for env in KNOBS:
            for k in ("QSB_NO_CKPT", "QSB_STAGP", "QSB_STAG", "QSB_NO_MERGE"):
                os.environ.pop(k, None)
            os.environ.update(env)
            try:
                v, g = qs.value_and_grad(h, prm)
                err = max(np.max(np.abs(np.array(g.d_betas) - db)), np.max(np.abs(np.array(g.d_gammas) - dg)))
                out.append(f"{env or 'default'}: {err:.1e}")
            except Exception as ex:  # noqa: BLE001
                out.append(f"{env}: {str(ex)[:60]}")
        print(f"n={n} p={p}: " + " | ".join(out), flush=True)
        h.close()
