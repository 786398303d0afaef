"""create_handle breakdown (context, precompute, |+> allocation, close) at small and
mid n, repeated -- the per-graph overhead of the many-graphs regime.
python tools/time_create.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import backend, costpoly

qs.create_handle(qs.maxcut_polynomial(qs.random_regular(12, 3, seed=1)), backend_name="b200").close()
for n in (8, 12, 16, 20, 24, 28):
    poly = qs.maxcut_polynomial(qs.random_regular(n, 3, seed=1))
    ts = []
    for rep in range(5):
        t0 = time.perf_counter()
        ctx = backend.create_context("b200")
        t1 = time.perf_counter()
        table = costpoly.precompute(poly, ctx)
        t2 = time.perf_counter()
        state = backend.alloc_plus_state(poly.n, ctx)
        ctx.synchronize()
        t3 = time.perf_counter()
        h = qs.circuit.SimHandle(poly, table, state, ctx)
        h.close()
        ctx.device.close()
        t4 = time.perf_counter()
        ts.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3))
    best = [min(x[i] for x in ts[1:]) * 1e3 for i in range(4)]
    print(f"n={n}: context {best[0]:.2f} ms, precompute {best[1]:.2f} ms, plus state {best[2]:.2f} ms, close {best[3]:.2f} ms")
