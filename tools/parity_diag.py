"""Parity diagnostics at ill-conditioned configs (SURVEY §8c rule, reading G22).

    python tools/parity_diag.py cfg sigma2,beta,nu lib1.so[,lib2.so...] [--dense K]

For each library build: strict failures (e > 1e-10 vs the FP64 oracle), failures of
SURVEY's κ rule with δ from ONE FP64 oracle run, and failures with δ = max over that
run and six FP64 replicas whose covariance entries are moved by up to ±2 ulp (the
spread of equally valid FP64 evaluations); plus the distribution of
ρ = |x_gpu − x_LD| / |x_or64 − x_LD| on the strict failures (ρ ≈ 1: the GPU is as
accurate as FP64 Alg. 1; ρ ≫ 1: it is not).  One JSON line per build."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bvgen  # noqa: E402
import oracle  # noqa: E402

cfg = sys.argv[1]
theta = tuple(float(x) for x in sys.argv[2].split(","))
libs = sys.argv[3].split(",")
p = bvgen.cached_plan(cfg)
c = bvgen.CONFIGS[cfg]["cfg"]
p = p.with_y(oracle.simulate_bv(p, theta, bvgen.normal(100 * c + 2, p.n)))
o64 = oracle.bv_loglik(p, theta)
old = oracle.bv_loglik(p, theta, long_double=True)
reps = [oracle.bv_loglik(p, theta, perturb_seed=2000 + s) for s in range(1, 7)]
l, _ = p.block_sizes()
s = np.abs(old["u"]) + np.abs(old["d"]) + l * 1.8378770664093456
import subprocess  # noqa: E402
oj = oracle.bv_loglik_joint(p, theta)  # diagnostic: a second exact FP64 formulation (joint Cholesky, CPU)


def grade(tag, d, u, ll):
    t = -0.5 * (u + d + l * 1.8378770664093456)
    strict = np.ones(len(l), bool)
    fail_1 = np.zeros(len(l), bool)
    fail_r = np.zeros(len(l), bool)
    rho = []
    for name, g in (("d", d), ("u", u), ("t", t)):
        e = np.abs(g - o64[name]) / s
        d1 = np.abs(o64[name] - old[name]) / s
        dr = d1.copy()
        for r in reps:
            dr = np.maximum(dr, np.abs(r[name] - old[name]) / s)
        eld = np.abs(g - old[name]) / s
        st = e <= 1e-10
        strict &= st
        fail_1 |= ~st & ~((d1 > 1e-11) & (eld <= 10 * d1))
        fail_r |= ~st & ~((dr > 1e-11) & (eld <= 10 * dr))
        rho.append(np.where(~st, eld / np.maximum(d1, 1e-300), 0.0))
    rho = np.max(np.stack(rho), axis=0)
    rr = rho[~strict]
    print(json.dumps({"cfg": cfg, "theta": theta, "impl": tag, "blocks": int(len(l)),
                      "strict_fail": int(np.sum(~strict)), "survey_rule_fail": int(fail_1.sum()),
                      "replica_rule_fail": int(fail_r.sum()),
                      "rho_median": float(np.median(rr)) if rr.size else 0.0,
                      "rho_p90": float(np.quantile(rr, 0.9)) if rr.size else 0.0,
                      "rho_max": float(rr.max()) if rr.size else 0.0,
                      "ll_rel_vs_fp64_oracle": abs(ll - o64["loglik"]) / abs(o64["loglik"]),
                      "ll_rel_vs_LD": abs(ll - old["loglik"]) / abs(old["loglik"]),
                      "fp64_oracle_ll_rel_vs_LD": abs(o64["loglik"] - old["loglik"]) / abs(old["loglik"])}))
    sys.stdout.flush()


grade("cpu_joint_fp64", oj["d"], oj["u"], oj["loglik"])
for lib in libs:
    # each build in its own process (one libbv per process)
    code = f"""
import sys, numpy as np
sys.path.insert(0, {ROOT!r})
import os
os.environ['BV_LIB_PATH'] = {os.path.abspath(lib)!r}
import bvgen, oracle
from paper_2410_04477_b200 import BlockVecchia
p = bvgen.cached_plan({cfg!r})
p = p.with_y(oracle.simulate_bv(p, {theta!r}, bvgen.normal({100 * c + 2}, p.n)))
ll, d, u = BlockVecchia(p).loglik_terms({theta!r})
np.save('/tmp/pd_d.npy', d); np.save('/tmp/pd_u.npy', u); print(repr(ll))
"""
    ll = float(subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True).stdout.split()[-1])
    d, u = np.load("/tmp/pd_d.npy"), np.load("/tmp/pd_u.npy")
    grade(os.path.basename(lib), d, u, ll)
