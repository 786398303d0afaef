"""Sharded E+grad on ONE GPU with virtual shards (the multi-GPU schedule; the swap is
device copies (per-position schedule) or fused stores (window chain)).
python tools/time_sharded.py n g p"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_13012_b200 as qs
from paper_2407_13012_b200 import dist

n, g, p = (int(x) for x in sys.argv[1:4])
poly = qs.maxcut_polynomial(qs.random_regular(n, 3 if n % 2 == 0 else 4, seed=1))
params = qs.linear_ramp_params(p)
sh = dist.ShardedHandle(poly, g, dist.VirtualExchanger(g))
for chain in ("1", "0"):
    os.environ["QSB_SHARD_CHAIN"] = chain
    sh.value_and_grad(params)
    sh.ctx.device.sync()
    t0 = time.perf_counter()
    for _ in range(3):
        v, dg, db = sh.value_and_grad(params)
    sh.ctx.device.sync()
    dt = (time.perf_counter() - t0) / 3
    dev = sh.ctx.device
    dev.prof_begin()
    sh.value_and_grad(params)
    prof = dev.prof_end()
    dev.sync()
    kinds = "  ".join(f"{k}={v[1]:.1f}ms/{int(v[0])}x/{v[2] / max(v[1], 1e-9) / 1e6:.0f}GB/s"
                      for k, v in sorted(prof.items()))
    print(f"n={n} g={g} p={p} {'window chain (fused swap)' if chain == '1' else 'per-position schedule + copy swap'}: "
          f"{1e3 * dt:.1f} ms per E+grad (all {1 << g} shards on one GPU)  E={v:.12f}\n    {kinds}")
sh.close()
