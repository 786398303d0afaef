"""Throughput of many small problems: one-by-one value_and_grad vs one batched launch.
python tools/time_batch.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import batch

suite = [g for _, g in qs.generate_suite(vertex_range=(6, 11), instances=40, seed=3)]
handles = [qs.create_handle(qs.maxcut_polynomial(g), backend_name="b200") for g in suite]
params = [qs.linear_ramp_params(6) for _ in handles]
batch.value_and_grad_batch(handles, params)
for _ in range(2):
    t0 = time.perf_counter()
    for h, p in zip(handles, params):
        qs.value_and_grad(h, p)
    t1 = time.perf_counter()
    batch.value_and_grad_batch(handles, params)
    t2 = time.perf_counter()
print(f"{len(handles)} graphs n=6..11 p=6 value_and_grad: one by one {1e3 * (t1 - t0):.1f} ms, "
      f"batched {1e3 * (t2 - t1):.2f} ms ({(t1 - t0) / (t2 - t1):.1f}x)")
