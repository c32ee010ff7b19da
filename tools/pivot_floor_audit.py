"""Audit of reading G15's non-PD floor (a pivot must exceed 1e-14·σ²) against SURVEY §8b's plain
"pivot ≤ 0", on the CPU oracle (set_pivot_floor):
  * the c2 MLE box: 60 seeded θ ~ log-U[0.05,5] × log-U[0.005,0.5] × U[0.2,3] on the c2 plan with
    y simulated at θ_true = (1, 0.052537, 1.5): how many θ change status, and how many blocks fail
    ONLY because of the floor (smallest pivot in (0, 1e-14·σ²]);
  * c3 at Table 1 β (1, 0.014290, 2.5): the same block counts;
  * the c2 MLE fit (paper_2410_04477_b200.mle.fit on the oracle's ℓ) under both rules: θ̂, ℓ̂.
Prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bvgen  # noqa: E402
import oracle  # noqa: E402
from paper_2410_04477_b200.mle import fit  # noqa: E402


def status(p, th, floor, k_range=None):
    oracle.set_pivot_floor(floor)
    try:
        oracle.bv_loglik(p, th, per_block=False, k_range=k_range)
        return 0, -1
    except oracle.OracleError as e:
        return e.status, e.failed_position


def floor_only_blocks(p, th):
    """Blocks failing with the floor but not with '≤ 0' (each block evaluated alone)."""
    n_floor, n_zero = 0, 0
    for k in range(p.bc):
        s1, _ = status(p, th, 1e-14, (k, k + 1))
        if s1:
            n_floor += 1
            s0, _ = status(p, th, 0.0, (k, k + 1))
            n_zero += 1 if s0 else 0
    return n_floor, n_zero


def main():
    out = {}
    th_true = (1.0, 0.052537, 1.5)
    p = bvgen.cached_plan("c2")
    p = p.with_y(oracle.simulate_bv(p, th_true, bvgen.normal(202, p.n)))
    u = bvgen.uniform(9001, 180).reshape(60, 3)
    thetas = [(float(np.exp(np.log(0.05) + u[i, 0] * np.log(100))), float(np.exp(np.log(0.005) + u[i, 1] * np.log(100))),
               float(0.2 + 2.8 * u[i, 2])) for i in range(60)]
    changed, fail_floor, fail_zero, blocks_floor_only = 0, 0, 0, 0
    for th in thetas:
        s1, k1 = status(p, th, 1e-14)
        s0, k0 = status(p, th, 0.0)
        fail_floor += s1 != 0
        fail_zero += s0 != 0
        if (s1, k1) != (s0, k0):
            changed += 1
        if s1:
            nf, nz = floor_only_blocks(p, th)
            blocks_floor_only += nf - nz
    out["c2_mle_box"] = {"thetas": 60, "non_pd_with_floor": int(fail_floor), "non_pd_with_le0": int(fail_zero),
                         "status_changed": int(changed), "blocks_failing_only_by_floor": int(blocks_floor_only)}
    c3 = bvgen.cached_plan("c3")
    th3 = (1.0, 0.014290, 2.5)
    c3 = c3.with_y(oracle.simulate_bv(c3, th3, bvgen.normal(302, c3.n)))
    s1, _ = status(c3, th3, 1e-14)
    s0, _ = status(c3, th3, 0.0)
    out["c3_table1"] = {"non_pd_with_floor": bool(s1), "non_pd_with_le0": bool(s0)}
    fits = {}
    for name, f in (("floor_1e-14", 1e-14), ("le_0", 0.0)):
        oracle.set_pivot_floor(f)
        r = fit(lambda th: oracle.bv_loglik(p, th, per_block=False)["loglik"])
        fits[name] = {"theta_hat": r["theta"], "loglik_hat": r["loglik"], "n_evals": r["n_evals"]}
    oracle.set_pivot_floor(1e-14)
    out["c2_mle_fit"] = fits
    print(json.dumps(out))


if __name__ == "__main__":
    main()
