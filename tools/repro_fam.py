"""Debug helper: one value_and_grad with a given sweep family (env) and size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2407_13012_b200 as qs
from conftest import random_instance

n, p = int(sys.argv[1]), int(sys.argv[2])
poly = random_instance(300 + n, n)
rs = np.random.default_rng(11 * n + p)
params = qs.QaoaParams(list(rs.uniform(-3.0, 3.0, p)), list(rs.uniform(-1.5, 1.5, p)))
h = qs.create_handle(poly, backend_name="b200")
v, g = qs.value_and_grad(h, params)
print("ok", v, g.d_betas, g.d_gammas)
