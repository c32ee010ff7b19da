"""Kernel time of one c2 evaluation at closed-form vs general ν (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bvgen
import paper_2410_04477_b200 as bvl
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
p = bvgen.cached_plan(cfg)
bv = bvl.BlockVecchia(p)
for nu in (1.5, 1.49, 1.0, 0.7, 2.2):
    for beta in (0.052537, 0.2, 0.01):
        th = (1.0, beta, nu)
        try:
            for _ in range(3):
                bv.loglik(th)
            t = time.perf_counter(); K = 10
            ks = []
            for _ in range(K):
                bv.loglik(th); ks.append(bv.last_kernel_ms())
            w = (time.perf_counter() - t) / K
            print(f"nu={nu} beta={beta}: kernel {min(ks):.3f} ms  wall {w*1e3:.3f} ms", flush=True)
        except Exception as e:
            print(nu, beta, "error", e)
