"""Where does one value_and_grad at n=16 spend its ~250 us?  python tools/prof_small_call.py"""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_13012_b200 as qs

poly = qs.maxcut_polynomial(qs.erdos_renyi(16, 0.5, seed=1))
h = qs.create_handle(poly, backend_name="b200")
params = qs.linear_ramp_params(6)
for _ in range(20):
    qs.value_and_grad(h, params)
t0 = time.perf_counter()
for _ in range(200):
    qs.value_and_grad(h, params)
print(f"value_and_grad n=16 p=6: {1e6 * (time.perf_counter() - t0) / 200:.1f} us per call")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    qs.value_and_grad(h, params)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
