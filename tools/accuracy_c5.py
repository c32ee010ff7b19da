"""c5's accuracy half (SURVEY §8d c5 row; PAPER.md:299-302 Eq. 6, :408): KL vs m and ℓ(θ)/n vs m.

    python tools/accuracy_c5.py > profiles/accuracy_r02.json

A tool, not a bench.py mode: it needs the oracle's block-Vecchia simulator for a model-distributed y
(test infrastructure; bench.py may touch oracle/ only in its CPU-baseline and reference legs).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bvgen  # noqa: E402

def main():
    """c5's accuracy half: KL(N0 ‖ N1) = ℓ0(θ; 0) − ℓa(θ; 0) (Eq. 6) at
    the reduced replica n = 20,000 / bc = 1,000 (l ≈ 20) for m ∈ {30, 60, 120, 200} — ℓa through
    bv_loglik with y = 0, ℓ0 the exact dense Gaussian log-likelihood (Eq. 1) at y = 0 by a dense FP64
    Cholesky (torch/cuSOLVER: the reference the paper takes from ExaGeoStat; checked
    against the oracle's exact_loglik at n = 4,000) — and ℓ(θ)/n against m at the full n = 2M (y
    simulated once with m_sim = 60)."""
    import torch
    import oracle
    import paper_2410_04477_b200 as bvl
    from paper_2410_04477_b200 import build as bvbuild
    torch.cuda.set_device(0)
    bvbuild.build()
    c = bvgen.CONFIGS["c5"]
    ms = [30, 60, 120, 200]
    out = {"metric": "block-Vecchia accuracy vs m (c5): KL divergence (Eq. 6) at n=20,000 and loglik/n at n=2M",
           "unit": "nats", "data": "synthetic", "dtype": "f64", "kl": {}, "loglik_per_n": {}}

    def exact_ll0(locs, theta):
        X = torch.from_numpy(locs).cuda()
        r = torch.cdist(X, X, compute_mode="donot_use_mm_for_euclid_dist") / theta[1]
        poly = {0.5: 1.0, 1.5: 1.0 + r, 2.5: 1.0 + r + r * r / 3.0}[theta[2]]
        S = theta[0] * poly * torch.exp(-r)
        del r
        L = torch.linalg.cholesky(S)
        ld = 2.0 * torch.log(torch.diagonal(L)).sum().item()
        del S, L
        torch.cuda.empty_cache()
        return -0.5 * (ld + locs.shape[0] * 1.8378770664093456)

    # pin the dense reference against the oracle's Eq. (1) at n = 4,000 (y = 0)
    th0 = tuple(c["theta"])
    loc4 = bvgen.locations(95, 4000, 2)
    e_or = oracle.exact_loglik(loc4, np.zeros(4000), th0)
    e_gpu = exact_ll0(loc4, th0)
    out["ll0_check_n4000"] = {"torch_dense": e_gpu, "oracle_exact": e_or, "rel": abs(e_gpu - e_or) / abs(e_or)}
    for theta in (th0, (1.0, 0.017512, 1.5)):
        key = f"theta={theta}"
        out["kl"][key] = {}
        kw = dict(n=20_000, bc=1_000, cfg=5)
        base = bvgen.make_plan("c5", m=30, **kw)
        ll0 = exact_ll0(base.locs, theta)
        for m in ms:
            p = bvgen.make_plan("c5", m=m, **kw).with_y(np.zeros(20_000))
            bv = bvl.BlockVecchia(p, device=0)
            lla = bv.loglik(theta)
            bv.close()
            out["kl"][key][str(m)] = {"kl": ll0 - lla, "ll0": ll0, "lla": lla}
    # ℓ(θ)/n vs m at full n
    theta = th0
    p60 = bvgen.cached_plan("c5", m=60)
    y = oracle.simulate_bv(p60, theta, bvgen.normal(502, p60.n))
    for m in ms:
        p = bvgen.cached_plan("c5", m=m).with_y(y)
        bv = bvl.BlockVecchia(p, device=0)
        ll = bv.loglik(theta)
        bv.close()
        out["loglik_per_n"][str(m)] = ll / p.n
    out["config"] = {"workload": "c5 accuracy: KL at n=20,000 bc=1,000 (theta of c5 and nu=1.5 secondary); "
                                 "loglik/n at n=2,000,000 bc=100,000 (y simulated with m_sim=60)", "m": ms}
    print(json.dumps(out))
    return 0



if __name__ == "__main__":
    main()
