"""Compare the general-ν pre-generation path with the in-kernel K_ν path at c2 over
random θ in the MLE box: count of θ whose ℓ / d_k / u_k differ bitwise, max relative ℓ gap."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bvgen  # noqa: E402
from paper_2410_04477_b200 import BlockVecchia  # noqa: E402

p = bvgen.cached_plan("c2")
p = p.with_y(bvgen.normal(7, p.n))
a = BlockVecchia(p)
os.environ["BV_NO_PREGEN"] = "1"
b = BlockVecchia(p)
rng = np.random.default_rng(3)
nd, worst = 0, 0.0
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 60):
    th = (rng.uniform(0.05, 5), rng.uniform(0.005, 0.5), rng.uniform(0.2, 3))
    try:
        la, da, ua = a.loglik_terms(th)
        lb, db, ub = b.loglik_terms(th)
    except Exception as e:  # noqa: BLE001
        print("theta", th, "error", e)
        continue
    same = la == lb and np.array_equal(da, db) and np.array_equal(ua, ub)
    if not same:
        nd += 1
        k = np.flatnonzero((da != db) | (ua != ub))
        worst = max(worst, abs(la - lb) / abs(lb))
        print("theta", th, "ll", la, lb, "blocks differing", len(k), "first", k[:5])
print("differing thetas", nd, "max rel ll gap", worst)
