"""compute-sanitizer target for the cost-table kernels: dyadic (subset-sum, incl.
mapped shard tables) and float (tiled term-order, > 2048 terms) builds, checked
against the oracle.  compute-sanitizer --tool racecheck python tools/san_tables.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import oracle
from paper_2407_13012_b200 import backend as be
from paper_2407_13012_b200.kernels import b200

ctx = be.create_context("b200")
r = np.random.default_rng(5)
n = 14
for kind, terms in (("dyadic", 300), ("float", 2500)):
    w = r.integers(-9, 10, terms).astype(np.float64) / 4 if kind == "dyadic" else r.normal(size=terms)
    m = np.array([int(x) & int(y) for x, y in zip(r.integers(0, 1 << n, terms), r.integers(0, 1 << n, terms))],
                 dtype=np.int64)
    out = b200.empty(ctx.device, 1 << n, np.float64)
    b200.build_cost_table(n, w, m, out)
    assert np.array_equal(np.asarray(out), oracle.precompute_table(w, m, n)), kind
    print(kind, "ok")
