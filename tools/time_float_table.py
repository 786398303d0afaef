"""Per-kind sweep times, integer (u16 compact + LUT) vs float (fp64 table + device
sincos) cost tables: weighted MaxCut K_n vs a dense QUBO, n (default 28), p=6,
value_and_grad, full vectors (QSB_NO_SYM=1) so only the table kind differs.
python tools/time_float_table.py [n]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("QSB_NO_SYM", "1")
import paper_2407_13012_b200 as qs
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
params = qs.linear_ramp_params(6)
for name, poly in (("wmaxcut_K%d" % n, bench.weighted_maxcut(n, 1)), ("qubo", bench.qubo_polynomial(n, 1))):
    h = qs.create_handle(poly, backend_name="b200")
    qs.value_and_grad(h, params)
    dev = h.ctx.device
    dev.sync()
    dev.prof_begin()
    t0 = time.perf_counter()
    for _ in range(3):
        qs.value_and_grad(h, params)
    dev.sync()
    ms = (time.perf_counter() - t0) / 3 * 1e3
    prof = dev.prof_end()
    print(f"{name}: {ms:.1f} ms per E+grad; " + ", ".join(f"{k} {v[1] / 3:.2f}" for k, v in sorted(prof.items())))
    h.close()
