"""One GPU, no sharding: E + gradient at n = 31 / 32 (180 GB of HBM3e holds ket + bra +
f64 table + compact index up to n = 32).  python tools/try_n32.py n"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = int(sys.argv[1])
os.environ["QAOA_MAX_QUBITS"] = str(n)
os.environ["QAOA_MEM_CEILING_BYTES"] = str(16 << n)
import paper_2407_13012_b200 as qs

poly = qs.maxcut_polynomial(qs.random_regular(n, 3, seed=1))
t0 = time.perf_counter()
h = qs.create_handle(poly, backend_name="b200")
h.ctx.synchronize()
t1 = time.perf_counter()
params = qs.linear_ramp_params(6)
v, g = qs.value_and_grad(h, params)
t2 = time.perf_counter()
v, g = qs.value_and_grad(h, params)
t3 = time.perf_counter()
print(f"n={n}: create_handle {t1 - t0:.2f} s, value_and_grad {1e3 * (t3 - t2):.0f} ms (first {1e3 * (t2 - t1):.0f} ms), "
      f"E={v:.12f}, |grad|max={max(abs(x) for x in g.d_betas + g.d_gammas):.6f}")
