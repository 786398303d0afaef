"""The paper's benchmark-suite regime end to end: problems.generate_suite(6..29, 5
instances per family and size; 580 graphs), p=6 linear ramp, one expectation +
gradient (value_and_grad) per graph.  Times (a) one handle at a time through the
public API and (b) batch.value_and_grad_batch per size (one launch for n <= 11,
concurrent streams for 12 <= n <= 22, one by one above), with create_handle
(precompute) timed separately.  Prints one JSON line.
python tools/time_suite.py [--hi 29]"""
import argparse
import json
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_13012_b200 as qs  # noqa: E402
from paper_2407_13012_b200 import batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--hi", type=int, default=29)
ap.add_argument("--threads", type=int, default=4)
args = ap.parse_args()
suite = qs.generate_suite(vertex_range=(6, args.hi), instances=5, seed=0)
by_n = defaultdict(list)
for fam, g in suite:
    by_n[g.num_vertices].append(qs.maxcut_polynomial(g))
params = qs.linear_ramp_params(6)
warm = qs.create_handle(by_n[16][0], backend_name="b200")
qs.value_and_grad(warm, params)
batch.value_and_grad_batch([warm], [params])
warm.close()
rows = {}
tot = defaultdict(float)
for n in sorted(by_n):
    polys = by_n[n]
    if n > 22:  # large registers: one handle at a time (25 x 2 x 16 * 2^n bytes would not fit)
        t_create = t_run = 0.0
        creates = []
        for poly in polys:
            t0 = time.perf_counter()
            h = qs.create_handle(poly, backend_name="b200")
            h.ctx.synchronize()
            t1 = time.perf_counter()
            qs.value_and_grad(h, params)
            t2 = time.perf_counter()
            h.close()
            t_create += t1 - t0
            t_run += t2 - t1
            creates.append(1e3 * (t1 - t0))
        rows[n] = {"graphs": len(polys), "create_ms": 1e3 * t_create, "one_by_one_ms": 1e3 * t_run,
                   "batched_ms": 1e3 * t_run, "create_median_ms": sorted(creates)[len(creates) // 2],
                   "create_max_ms": max(creates)}
    else:
        t0 = time.perf_counter()
        hs = [qs.create_handle(p, backend_name="b200") for p in polys]
        for h in hs:
            h.ctx.synchronize()
        t1 = time.perf_counter()
        first = [qs.value_and_grad(h, params) for h in hs]  # first calls allocate each handle's bra
        t2a = time.perf_counter()
        one = [qs.value_and_grad(h, params) for h in hs]
        t2 = time.perf_counter()
        assert first == one
        bat = batch.value_and_grad_batch(hs, [params] * len(hs), threads=args.threads)
        t3 = time.perf_counter()
        for (va, ga), (vb, gb) in zip(one, bat):  # equal to rounding (checkpointed vs batched walk)
            assert abs(va - vb) <= 1e-12 * max(1.0, abs(va)), n
            assert max(abs(x - y) for x, y in zip(ga.d_betas + ga.d_gammas, gb.d_betas + gb.d_gammas)) <= \
                1e-12 * max(1.0, max(abs(x) for x in ga.d_betas + ga.d_gammas)), n
        for h in hs:
            h.close()
        rows[n] = {"graphs": len(hs), "create_ms": 1e3 * (t1 - t0), "first_call_ms": 1e3 * (t2a - t1),
                   "one_by_one_ms": 1e3 * (t2 - t2a), "batched_ms": 1e3 * (t3 - t2)}
    for k in ("create_ms", "one_by_one_ms", "batched_ms"):
        tot[k] += rows[n][k]
    tot["graphs"] += len(polys)
mid = {k: sum(rows[n][k] for n in rows if 12 <= n <= 22) for k in ("one_by_one_ms", "batched_ms")}
small = {k: sum(rows[n][k] for n in rows if n <= 11) for k in ("one_by_one_ms", "batched_ms")}
print(json.dumps({"suite": f"generate_suite(6..{args.hi}, instances=5, seed=0), p=6 ramp, value_and_grad per graph",
                  "totals": dict(tot), "n_le_11": small, "n_12_22": mid,
                  "speedup_total": tot["one_by_one_ms"] / tot["batched_ms"],
                  "speedup_12_22": mid["one_by_one_ms"] / mid["batched_ms"],
                  "per_n": rows}))
