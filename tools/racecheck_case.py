import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2407_13012_b200 as qs
from conftest import random_instance
n = int(sys.argv[1])
poly = random_instance(99 + n, n)
h = qs.create_handle(poly, backend_name="b200")
params = qs.QaoaParams([0.3, -0.5, 0.7], [0.9, 0.2, -0.4])
v, g = qs.value_and_grad(h, params)
print("n", n, "v", v)
