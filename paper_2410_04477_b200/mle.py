"""Maximum-likelihood fit of θ = (σ², β, ν) over the block-Vecchia ℓ(θ) — the c2 workload.

The paper maximises ℓ with NLopt's BOBYQA, a bound-constrained derivative-free
method, estimating all three of (σ², β, ν) (NLopt 2.7.1 at
PAPER.md:284).  BOBYQA itself is not in this image; any bounded derivative-free
method is admissible for the harness, so this driver runs
scipy's bounded Nelder–Mead simplex search in log(σ²), log(β), ν (on the
strongly correlated (σ², β) ridge of the Matérn likelihood it needs ~5× fewer
evaluations than bounded Powell: 225 vs 1096 on tests/test_mle.py's plan).  Host-only: every ℓ(θ) is
one call of the library (`BlockVecchia.loglik`, i.e. `bv_loglik`) or of any
callable with the same signature.  A non-positive-definite θ scores −∞
(SURVEY §8d c2 recipe).

    from paper_2410_04477_b200 import BlockVecchia
    from paper_2410_04477_b200.mle import fit
    res = fit(BlockVecchia(plan).loglik)          # start (0.5, 0.1, 1.0), box of SURVEY §8d

Under multi-GPU every rank runs this redundantly: ℓ is bitwise identical on all
ranks (exact fixed-point sum), so they propose the same θ sequence.
"""
from __future__ import annotations

import math
import time

import numpy as np

NOT_PD = 3  # BV_ENOTPD (include/bv.h); the oracle reports non-PD with the same status

THETA0 = (0.5, 0.1, 1.0)
BOUNDS = ((0.05, 5.0), (0.005, 0.5), (0.2, 3.0))


def fit(loglik, theta0=THETA0, bounds=BOUNDS, max_evals: int = 2000, rtol: float = 1e-7, fix_nu=None):
    """Maximise loglik(θ) over the box; returns a dict with theta, loglik, n_evals, wall_s, trace.

    Stops when the simplex's spread of ℓ falls below rtol·|ℓ(θ0)| (and its spread in
    x below 1e-7) or after max_evals evaluations.  fix_nu: estimate (σ², β) only, at that ν.
    """
    from scipy.optimize import minimize

    trace = []

    def to_theta(x):
        s2, b = math.exp(x[0]), math.exp(x[1])
        nu = fix_nu if fix_nu is not None else float(x[2])
        return (s2, b, nu)

    def f(x):
        th = to_theta(x)
        try:
            v = loglik(th)
        except Exception as e:  # NOT_PD (status 3 in the library and the oracle alike) → −∞;
            if getattr(e, "status", None) != NOT_PD:  # any other status (EINVAL, ECUDA, ENCCL, ...) is raised
                raise
            v = -math.inf
        trace.append((th, v))
        return 1e300 if not math.isfinite(v) else -v

    lo = [math.log(bounds[0][0]), math.log(bounds[1][0])]
    hi = [math.log(bounds[0][1]), math.log(bounds[1][1])]
    x0 = [math.log(theta0[0]), math.log(theta0[1])]
    if fix_nu is None:
        lo.append(bounds[2][0])
        hi.append(bounds[2][1])
        x0.append(theta0[2])
    t0 = time.perf_counter()
    fscale = f(np.array(x0))
    fatol = rtol * (abs(fscale) if fscale < 1e300 else 1.0)
    r = minimize(f, np.array(x0), method="Nelder-Mead", bounds=list(zip(lo, hi)),
                 options={"maxfev": max_evals - 1, "fatol": fatol, "xatol": 1e-7})
    wall = time.perf_counter() - t0
    best = max((t for t in trace if math.isfinite(t[1])), key=lambda t: t[1], default=(to_theta(r.x), -math.inf))
    return {"theta": tuple(float(v) for v in best[0]), "loglik": float(best[1]), "n_evals": len(trace),
            "wall_s": wall, "evals_per_s": len(trace) / wall if wall > 0 else math.inf,
            "converged": bool(r.success), "message": str(r.message), "trace": trace}
