"""Cost-table build times: the default path (exact int64 subset-sum for dyadic weights,
the tiled term-order kernel otherwise) against the tiled kernel (QSB_NO_ZETA=1) and the
per-x kernel (QSB_NO_ZETA=2), and create_handle end to end.

    python tools/time_precompute.py [--max-n 32]

Prints one line per (problem, n): precompute+finish (qsb_table_create) in ms for both
kernels, whether the tables are bit-identical, and create_handle wall time."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import backend as be
from paper_2407_13012_b200.kernels import b200

ap = argparse.ArgumentParser()
ap.add_argument("--max-n", type=int, default=32)
ap.add_argument("--only", default=None, help="comma list of problem names")
args = ap.parse_args()

ctx = be.create_context("b200")


def build(poly, out):
    ctx.synchronize()
    t0 = time.perf_counter()
    b200.build_cost_table(poly.n, poly.weights, poly.masks, out)
    ctx.synchronize()
    return 1e3 * (time.perf_counter() - t0)


cases = [("reg3", n, lambda n: qs.maxcut_polynomial(qs.random_regular(n, 3, seed=1))) for n in (24, 28, 30)]
cases += [("er0.5", n, lambda n: qs.maxcut_polynomial(qs.erdos_renyi(n, 0.5, seed=1))) for n in (24, 29)]
cases += [("wK", n, lambda n: bench.weighted_maxcut(n, 1)) for n in (28, 32)]
cases += [("qubo(float)", n, lambda n: bench.qubo_polynomial(n, 1)) for n in (28, 32)]
os.environ.setdefault("QAOA_MAX_QUBITS", "34")
os.environ.setdefault("QAOA_MEM_CEILING_BYTES", str(16 << 32))
for name, n, mk in cases:
    if n > args.max_n or (args.only and name not in args.only.split(",")):
        continue
    poly = mk(n)
    out = b200.empty(ctx.device, 1 << n, np.float64)
    build(poly, out)  # warm-up (allocation of the compact index etc.)
    t_fast = min(build(poly, out) for _ in range(2))
    a = np.asarray(out) if n <= 30 else None
    os.environ["QSB_NO_ZETA"] = "1"
    t_tiled = min(build(poly, out) for _ in range(2))
    same1 = bool(np.array_equal(a, np.asarray(out))) if a is not None else None
    os.environ["QSB_NO_ZETA"] = "2"
    t_slow = min(build(poly, out) for _ in range(2))
    del os.environ["QSB_NO_ZETA"]
    same = (same1 and bool(np.array_equal(a, np.asarray(out)))) if a is not None else "n/a (n>30: not copied)"
    out.free()
    t0 = time.perf_counter()
    h = qs.create_handle(poly, backend_name="b200")
    h.ctx.synchronize()
    t_create = 1e3 * (time.perf_counter() - t0)
    h.close()
    print(f"{name:12s} n={n:2d} terms={poly.num_terms:5d}: table {t_fast:9.2f} ms (tiled term-order kernel "
          f"{t_tiled:9.2f} ms, per-x kernel {t_slow:9.2f} ms, "
          f"identical={same}); create_handle {t_create:9.2f} ms", flush=True)
