"""The parity rule (DESIGN.md §3 G21/G22) shared by the GPU tests.

For each block i and x ∈ {d_i, u_i, t_i}, with the scale
s_i = |u_i| + |d_i| + l_i log 2π (G21: d and t can cross zero):
    e_i = |x_gpu − x_or64| / s_i          GPU vs the FP64 oracle
    δ_i = max_r |x_r − x_orLD| / s_i      FP64's own error vs the 80-bit oracle,
          r over the FP64 oracle and six replicas whose covariance entries are
          moved by up to ±2 ulp (oracle perturb_seed 2001..2006; an FP64
          Eq. (7) evaluation is a few roundings): one FP64 run is a single
          noisy sample of that error, the spread over equally valid roundings
          is its size (G22; tools/kappa_diag.py shows the GPU/δ ratio has
          median ≈ 0.5, i.e. the GPU is as accurate as FP64 Alg. 1)
A block passes if e_i ≤ 1e-10 (BASELINE.json north_star), or — only where
FP64 itself is that far off (δ_i > 1e-11, ill-conditioned blocks, G22) — if
|x_gpu − x_orLD| / s_i ≤ 10·δ_i.  ℓ: |ℓ_gpu − ℓ_or| ≤ 1e-9·|ℓ_or| (north_star).
"""
import math

import numpy as np

LN2PI = 1.8378770664093456
TOL_BLOCK = 1e-10
TOL_LL = 1e-9


def compare(gpu_d, gpu_u, ora64, oraLD, l, gpu_ll=None, ora_ll=None, label="", replicas=()):
    """Assert the parity rule; return a summary dict (max e, κ-branch count).

    ``replicas``: extra FP64 oracle runs (perturb_seed ≠ 0) for δ."""
    l = np.asarray(l, dtype=np.float64)
    s = np.abs(oraLD["u"]) + np.abs(oraLD["d"]) + l * LN2PI
    gpu_t = -0.5 * (gpu_u + gpu_d + l * LN2PI)
    worst = 0.0
    kappa_used = 0
    fails = []
    for name, g, o64, old in (("d", gpu_d, ora64["d"], oraLD["d"]), ("u", gpu_u, ora64["u"], oraLD["u"]),
                              ("t", gpu_t, ora64["t"], oraLD["t"])):
        e = np.abs(g - o64) / s
        delta = np.abs(o64 - old) / s
        for rep in replicas:
            xr = rep[name] if name != "t" else rep["t"]
            delta = np.maximum(delta, np.abs(xr - old) / s)
        eld = np.abs(g - old) / s
        ok_strict = e <= TOL_BLOCK
        ok_kappa = (delta > 1e-11) & (eld <= 10 * delta)
        ok = ok_strict | ok_kappa
        kappa_used += int(np.sum(~ok_strict & ok_kappa))
        worst = max(worst, float(e.max()) if e.size else 0.0)
        if not ok.all():
            bad = np.where(~ok)[0]
            fails.append((name, bad[:10].tolist(), e[bad[:10]].tolist(), delta[bad[:10]].tolist()))
    assert not fails, f"{label}: blocks failing parity: {fails}"
    out = {"blocks": int(len(l)), "max_e": worst, "kappa_branch": kappa_used,
           "median_e": float(np.median(np.abs(gpu_t - ora64["t"]) / s)) if len(l) else 0.0}
    if gpu_ll is not None and ora_ll is not None:
        rel = abs(gpu_ll - ora_ll) / abs(ora_ll)
        out["ll_rel"] = rel
        assert rel <= TOL_LL, f"{label}: loglik rel err {rel:.3e} (gpu {gpu_ll!r}, oracle {ora_ll!r})"
    return out
