"""One value_and_grad (p=3) through the window chain, the target of compute-sanitizer
runs: python tools/racecheck_case.py N [qubo]  (qubo: dense float-weight table -> the
staged fp64 table tiles; N >= 21 MaxCut-like instances run Z2-reduced with forward
checkpoints)"""
import sys, os
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE)); sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))
import numpy as np
import paper_2407_13012_b200 as qs
from conftest import random_instance
n = int(sys.argv[1])
if len(sys.argv) > 2 and sys.argv[2] == "qubo":
    rs = np.random.default_rng(n)
    terms = [((rs.random() - 0.5) * 8.0, 1 << i) for i in range(n)]
    terms += [((rs.random() - 0.5) * 8.0, (1 << i) | (1 << j)) for i in range(n) for j in range(i + 1, n) if rs.random() < 0.3]
    poly = qs.Polynomial(n, terms)
else:
    poly = random_instance(99 + n, n)
h = qs.create_handle(poly, backend_name="b200")
params = qs.QaoaParams([0.3, -0.5, 0.7], [0.9, 0.2, -0.4])
v, g = qs.value_and_grad(h, params)
print("n", n, "v", v)
