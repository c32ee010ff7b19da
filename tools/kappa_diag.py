"""Parity diagnostics at ill-conditioned configs: distribution of
|x_gpu − x_LD| / δ where δ is the FP64 oracle's own error (max over entry-
perturbed replicas).  perturb_seed s < 1000: ±1 ulp; s = 1000·w + i: ±w ulp."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import bvgen  # noqa: E402
import oracle  # noqa: E402
from paper_2410_04477_b200 import BlockVecchia  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
theta = tuple(float(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 else (1.0, 0.014290, 2.5)
p = bvgen.cached_plan(cfg)
c = bvgen.CONFIGS[cfg]["cfg"]
p = p.with_y(oracle.simulate_bv(p, theta, bvgen.normal(100 * c + 2, p.n)))
ll, d, u = BlockVecchia(p).loglik_terms(theta)
o64 = oracle.bv_loglik(p, theta)
old = oracle.bv_loglik(p, theta, long_double=True)
l, _ = p.block_sizes()
s = np.abs(old["u"]) + np.abs(old["d"]) + l * 1.8378770664093456
for label, seeds in (("1ulp x3", (1, 2, 3)), ("1ulp x6", (1, 2, 3, 4, 5, 6)), ("2ulp x3", (2001, 2002, 2003)),
                     ("2ulp x6", (2001, 2002, 2003, 2004, 2005, 2006))):
    reps = [oracle.bv_loglik(p, theta, perturb_seed=sd) for sd in seeds]
    for name, g, o in (("d", d, o64["d"]), ("u", u, o64["u"])):
        delta = np.abs(o - old[name]) / s
        for r in reps:
            delta = np.maximum(delta, np.abs(r[name] - old[name]) / s)
        eld = np.abs(g - old[name]) / s
        e = np.abs(g - o) / s
        strict = e <= 1e-10
        ratio = eld / np.maximum(delta, 1e-300)
        bad = (~strict) & ~((delta > 1e-11) & (ratio <= 10))
        print(f"{cfg} {label} {name}: strict-fail {np.sum(~strict)}, kappa-fail {np.sum(bad)}, "
              f"ratio p50 {np.median(ratio[~strict]) if np.any(~strict) else 0:.2f} "
              f"p99 {np.percentile(ratio[~strict], 99) if np.any(~strict) else 0:.2f} max {ratio[~strict].max() if np.any(~strict) else 0:.2f}")
print("ll rel", abs(ll - o64["loglik"]) / abs(o64["loglik"]))
