"""create_handle / value_and_grad / close per graph, one at a time, printing each create
time (the suite's large-n loop): python tools/time_create_loop.py N1,N2,.. [count]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_13012_b200 as qs

ns = [int(x) for x in sys.argv[1].split(",")]
count = int(sys.argv[2]) if len(sys.argv) > 2 else 6
params = qs.linear_ramp_params(6)
w = qs.create_handle(qs.maxcut_polynomial(qs.random_regular(16, 3, seed=1)), backend_name="b200")
qs.value_and_grad(w, params)
w.close()
for n in ns:
  out = []
  for s in range(count):
    poly = qs.maxcut_polynomial(qs.erdos_renyi(n, 0.5, seed=s))
    t0 = time.perf_counter()
    h = qs.create_handle(poly, backend_name="b200")
    h.ctx.synchronize()
    t1 = time.perf_counter()
    qs.value_and_grad(h, params)
    t2 = time.perf_counter()
    h.close()
    t3 = time.perf_counter()
    out.append(f"create {1e3 * (t1 - t0):7.2f} E+grad {1e3 * (t2 - t1):7.2f} close {1e3 * (t3 - t2):6.2f}")
  print(f"n={n} BIGCACHE={'off' if os.environ.get('QSB_NO_BIGCACHE') == '1' else 'on'}: " + " | ".join(out), flush=True)
