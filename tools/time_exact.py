"""Exact mode (QAOA_B200_EXACT=1, bit-identical to the reference) timings.  python tools/time_exact.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["QAOA_B200_EXACT"] = "1"
import paper_2407_13012_b200 as qs

for name, poly, p in (("C2 er24 p4", qs.maxcut_polynomial(qs.erdos_renyi(24, 0.5, seed=1)), 4),
                      ("C3 reg3 n30 p6", qs.maxcut_polynomial(qs.random_regular(30, 3, seed=1)), 6)):
    h = qs.create_handle(poly, backend_name="b200")
    params = qs.linear_ramp_params(p)
    qs.expectation(h, params)
    t0 = time.perf_counter()
    e = qs.expectation(h, params)
    t1 = time.perf_counter()
    g = qs.gradient(h, params)
    t2 = time.perf_counter()
    print(f"exact {name}: expectation {1e3 * (t1 - t0):.1f} ms (E={e!r}), gradient {1e3 * (t2 - t1):.1f} ms")
    h.close()
