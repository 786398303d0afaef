"""Wall time of value_and_grad / expectation for small registers (p=6 random angles)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2407_13012_b200 as qs

p = 6
rs = np.random.default_rng(0)
params = qs.QaoaParams(list(rs.uniform(-1, 1, p)), list(rs.uniform(-1, 1, p)))
for n in [6, 8, 10, 11, 12, 14, 16, 18, 20, 22]:
    poly = qs.maxcut_polynomial(qs.erdos_renyi(n, 0.5, seed=1))
    h = qs.create_handle(poly, backend_name="b200")
    for _ in range(3):
        qs.value_and_grad(h, params)
    reps = 50 if n <= 20 else 10
    t0 = time.perf_counter()
    for _ in range(reps):
        qs.value_and_grad(h, params)
    t1 = time.perf_counter()
    for _ in range(reps):
        qs.expectation(h, params)
    t2 = time.perf_counter()
    launches0 = h.ctx.device.launches()
    qs.value_and_grad(h, params)
    nl = h.ctx.device.launches() - launches0
    print(f"n={n:2d}  value_and_grad {1e6 * (t1 - t0) / reps:9.1f} us  expectation {1e6 * (t2 - t1) / reps:9.1f} us  "
          f"launches/E+grad {nl}")
    h.close()
