"""Where does a 10^6-shot draw at n=30 spend its time (C3)?  python tools/time_sample.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_13012_b200 as qs

h = qs.create_handle(qs.maxcut_polynomial(qs.random_regular(30, 3, seed=1)), backend_name="b200")
params = qs.linear_ramp_params(6)
dev = h.ctx.device
for rep in range(3):
    qs.simulate(h, params)
    dev.sync()
    t0 = time.perf_counter()
    d = h.state.data  # mirror expansion (Z2) if pending
    dev.sync()
    t1 = time.perf_counter()
    ss = qs.draw(h, 1_000_000, 1)
    t2 = time.perf_counter()
    print(f"rep {rep}: mirror {1e3 * (t1 - t0):.2f} ms, draw {1e3 * (t2 - t1):.2f} ms, pending={h.state._pending}")
