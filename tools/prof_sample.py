"""Time qs.draw at C3 (n=30, p=6 ramp, 10^6 shots) by phase: python tools/prof_sample.py [n] [shots]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_13012_b200 as qs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
shots = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
poly = qs.maxcut_polynomial(qs.random_regular(n, 3, seed=1))
h = qs.create_handle(poly, backend_name="b200")
qs.simulate(h, qs.linear_ramp_params(6))
h.ctx.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    ss = qs.draw(h, shots, 1)
    t1 = time.perf_counter()
    print(f"draw {shots} shots: {1e3 * (t1 - t0):.2f} ms  best {qs.best_of(ss)}")
