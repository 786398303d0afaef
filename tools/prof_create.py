"""Where does create_handle's wall time go at n=30?  python tools/prof_create.py"""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_13012_b200 as qs

poly = qs.maxcut_polynomial(qs.random_regular(30, 3, seed=1))
h0 = qs.create_handle(qs.maxcut_polynomial(qs.random_regular(12, 3, seed=1)), backend_name="b200")  # CUDA init
h0.close()
for rep in range(2):
    t0 = time.perf_counter()
    pr = cProfile.Profile()
    pr.enable()
    h = qs.create_handle(poly, backend_name="b200")
    h.ctx.synchronize()
    pr.disable()
    print(f"create_handle n=30: {time.perf_counter() - t0:.3f} s")
    h.close()
pstats.Stats(pr).sort_stats("cumulative").print_stats(15)
