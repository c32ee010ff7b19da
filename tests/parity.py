"""The parity rule (DESIGN.md §3 G21/G22) shared by the GPU tests.

For each block i and x ∈ {d_i, u_i, t_i}, with the scale
s_i = |u_i| + |d_i| + l_i log 2π (G21: d and t can cross zero):
    e_i = |x_gpu − x_or64| / s_i          GPU vs the FP64 oracle
    δ_i = |x_or64 − x_orLD| / s_i         FP64's own error: ONE FP64 oracle run vs
                                          the 80-bit oracle (exactly)
A block passes if e_i ≤ 1e-10 (BASELINE.json north_star), or — only where FP64
itself is that far off (δ_i > 1e-11, ill-conditioned blocks, G22) — if
|x_gpu − x_orLD| / s_i ≤ 10·δ_i (the GPU is no worse than 10× the FP64
oracle's own error).  ℓ: |ℓ_gpu − ℓ_or| ≤ 1e-9·|ℓ_or| (north_star).

Where a block misses this rule, its δ is re-measured as the spread of SEVEN
equally valid FP64 evaluations (the FP64 oracle and six replicas whose
covariance entries are moved by up to ±2 ulp, oracle perturb_seed 2001..2006):
one FP64 run is a single sample of FP64's own error, and at κ ≈ 1e10-1e12 a
lucky sample can sit far below it.  Such a block counts as a "replica
exception"; the count is reported and bounded per case (G22 and
profiles/parity_r02.md give the evidence: at c3's Table 1 β a plain CPU FP64
joint-Cholesky formulation misses the single-run rule on 3.3 % of blocks, the
GPU on 5.8 %, and both pass the replica rule everywhere).  A block that misses
both fails the test.

Every comparison reports ("every report states how many blocks
used the κ branch", "report e_i's distribution"): blocks checked, strict
failures (e > 1e-10), κ-branch count, replica exceptions, e median / p99 /
max, ℓ relative error.
With BV_PARITY_REPORT=<file> set, each report is appended there as one JSON
line (tools/parity_report.py turns the file into profiles/parity_r02.md).
"""
import json
import os

import numpy as np

LN2PI = 1.8378770664093456
TOL_BLOCK = 1e-10
TOL_LL = 1e-9


def _emit(rec):
    path = os.environ.get("BV_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")
    print("parity", json.dumps(rec))


def compare(gpu_d, gpu_u, ora64, oraLD, l, gpu_ll=None, ora_ll=None, label="", theta=None, strict_only=False,
            replicas=None, max_exceptions=0):
    """Assert the parity rule on every block given; return (and report) the summary.

    ``oraLD`` is the 80-bit oracle on the same positions (None with ``strict_only``:
    then every block must pass e ≤ 1e-10).  ``replicas``: a callable returning the six
    perturbed FP64 oracle runs on the same positions (called only if some block misses the
    single-run rule); at most ``max_exceptions`` blocks may pass by the replica δ alone."""
    l = np.asarray(l, dtype=np.float64)
    ref = oraLD if oraLD is not None else ora64
    s = np.abs(ref["u"]) + np.abs(ref["d"]) + l * LN2PI
    gpu_t = -0.5 * (gpu_u + gpu_d + l * LN2PI)
    e_blk = np.zeros(len(l))
    strict_blk = np.ones(len(l), dtype=bool)
    ok_blk = np.ones(len(l), dtype=bool)
    ok_rep = np.ones(len(l), dtype=bool)
    reps = None
    for name, g, o64 in (("d", gpu_d, ora64["d"]), ("u", gpu_u, ora64["u"]), ("t", gpu_t, ora64["t"])):
        e = np.abs(g - o64) / s
        e_blk = np.maximum(e_blk, e)
        ok_strict = e <= TOL_BLOCK
        if oraLD is not None and not strict_only:
            old = oraLD[name]
            delta = np.abs(o64 - old) / s
            eld = np.abs(g - old) / s
            ok = ok_strict | ((delta > 1e-11) & (eld <= 10 * delta))
            okr = ok.copy()
            if not ok.all() and replicas is not None:
                reps = reps if reps is not None else replicas()
                dr = delta.copy()
                for r in reps:
                    dr = np.maximum(dr, np.abs(r[name] - old) / s)
                okr = ok_strict | ((dr > 1e-11) & (eld <= 10 * dr))
        else:
            ok = okr = ok_strict
        strict_blk &= ok_strict
        ok_blk &= ok
        ok_rep &= okr
    exc = ~ok_blk & ok_rep
    bad = np.where(~ok_rep)[0]
    rec = {"label": label, "theta": list(theta) if theta is not None else None, "blocks": int(len(l)),
           "strict_fail": int(np.sum(~strict_blk)), "kappa_branch": int(np.sum(~strict_blk & ok_blk)),
           "replica_exceptions": int(np.sum(exc)), "failed": int(len(bad)),
           "e_median": float(np.median(e_blk)) if len(l) else 0.0,
           "e_p99": float(np.quantile(e_blk, 0.99)) if len(l) else 0.0,
           "e_max": float(e_blk.max()) if len(l) else 0.0}
    if gpu_ll is not None and ora_ll is not None:
        rec["ll_rel"] = abs(gpu_ll - ora_ll) / abs(ora_ll)
    _emit(rec)
    assert len(bad) == 0, f"{label}: blocks failing parity: {bad[:10].tolist()} (e {e_blk[bad[:10]].tolist()})"
    assert rec["replica_exceptions"] <= max_exceptions, rec
    if "ll_rel" in rec:
        assert rec["ll_rel"] <= TOL_LL, f"{label}: loglik rel err {rec['ll_rel']:.3e} (gpu {gpu_ll!r}, oracle {ora_ll!r})"
    return rec


def compare_all_strict_then_ld(plan, theta, gpu_d, gpu_u, o64, label, gpu_ll=None, max_ld=400, max_exceptions=0):
    """Every position: e ≤ 1e-10 against the FP64 oracle; the 80-bit oracle (κ branch) runs only on
    the positions that miss it (at most max_ld of them, else the case fails), the replica δ only on
    those that miss the single-run rule too."""
    import oracle
    l, _ = plan.block_sizes()
    l = np.asarray(l, dtype=np.float64)
    s = np.abs(o64["u"]) + np.abs(o64["d"]) + l * LN2PI
    gpu_t = -0.5 * (gpu_u + gpu_d + l * LN2PI)
    e_blk = np.maximum.reduce([np.abs(gpu_d - o64["d"]) / s, np.abs(gpu_u - o64["u"]) / s,
                               np.abs(gpu_t - o64["t"]) / s])
    miss = np.where(e_blk > TOL_BLOCK)[0]
    assert len(miss) <= max_ld, f"{label}: {len(miss)} blocks miss 1e-10 (more than {max_ld})"
    bad, exc = [], []
    whole = len(miss) > 100  # many misses: one whole-range 80-bit run instead of one per position
    old_all = oracle.bv_loglik(plan, theta, long_double=True) if whole else None
    reps_all = None
    for k in miss:
        kr = (int(k), int(k) + 1)
        old = ({n: old_all[n][k:k + 1] for n in ("d", "u", "t")} if whole else
               oracle.bv_loglik(plan, theta, long_double=True, k_range=kr))
        reps = None
        for name, g in (("d", gpu_d[k]), ("u", gpu_u[k]), ("t", gpu_t[k])):
            delta = abs(o64[name][k] - old[name][0]) / s[k]
            eld = abs(g - old[name][0]) / s[k]
            if abs(g - o64[name][k]) / s[k] > TOL_BLOCK and not (delta > 1e-11 and eld <= 10 * delta):
                if reps is None:
                    if whole:
                        reps_all = reps_all or [oracle.bv_loglik(plan, theta, perturb_seed=2000 + q) for q in range(1, 7)]
                        reps = [{n: r[n][k:k + 1] for n in ("d", "u", "t")} for r in reps_all]
                    else:
                        reps = [oracle.bv_loglik(plan, theta, k_range=kr, perturb_seed=2000 + q) for q in range(1, 7)]
                dr = max([delta] + [abs(r[name][0] - old[name][0]) / s[k] for r in reps])
                (exc if (dr > 1e-11 and eld <= 10 * dr) else bad).append((int(k), name, float(delta), float(eld)))
    nbad = len({b[0] for b in bad})
    nexc = len({b[0] for b in exc} - {b[0] for b in bad})
    rec = {"label": label, "theta": list(theta), "blocks": int(len(l)), "strict_fail": int(len(miss)),
           "kappa_branch": int(len(miss) - nbad - nexc), "replica_exceptions": int(nexc), "failed": int(nbad),
           "e_median": float(np.median(e_blk)), "e_p99": float(np.quantile(e_blk, 0.99)),
           "e_max": float(e_blk.max())}
    if gpu_ll is not None:
        rec["ll_rel"] = abs(gpu_ll - o64["loglik"]) / abs(o64["loglik"])
    _emit(rec)
    assert not bad, f"{label}: blocks failing parity: {bad[:10]}"
    assert nexc <= max_exceptions, rec
    if gpu_ll is not None:
        assert rec["ll_rel"] <= TOL_LL, rec
    return rec
