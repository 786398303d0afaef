"""Unsharded E+grad wall time on one GPU (the comparison row of tools/time_sharded.py):
python tools/time_unsharded.py n p  (QSB_NO_SYM=1 / QSB_NO_CKPT=1 select the variants)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_13012_b200 as qs

n, p = int(sys.argv[1]), int(sys.argv[2])
os.environ.setdefault("QAOA_MAX_QUBITS", str(max(30, n)))
os.environ.setdefault("QAOA_MEM_CEILING_BYTES", str(max(16 << 30, 40 << n)))
h = qs.create_handle(qs.maxcut_polynomial(qs.random_regular(n, 3 if n % 2 == 0 else 4, seed=1)), backend_name="b200")
params = qs.linear_ramp_params(p)
qs.value_and_grad(h, params)
h.ctx.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    v, g = qs.value_and_grad(h, params)
h.ctx.synchronize()
dt = (time.perf_counter() - t0) / 3
dev = h.ctx.device
dev.prof_begin()
qs.value_and_grad(h, params)
prof = dev.prof_end()
kinds = "  ".join(f"{k}={v[1]:.1f}ms/{int(v[0])}x/{v[2] / max(v[1], 1e-9) / 1e6:.0f}GB/s" for k, v in sorted(prof.items()))
env = " ".join(f"{k}={os.environ[k]}" for k in ("QSB_NO_SYM", "QSB_NO_CKPT") if k in os.environ) or "default"
print(f"n={n} p={p} unsharded [{env}]: {1e3 * dt:.1f} ms per E+grad  E={v:.12f}\n    {kinds}")
