"""Block Vecchia vs classic Vecchia (bc = n) at n = 20k (§3.2 setting): device time per evaluation."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bvgen
import paper_2410_04477_b200 as bvl
theta = (1.0, 0.052537, 1.5)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
for bc, m in [(n, 30), (n, 60), (1500, 30), (1500, 60), (1500, 120), (1500, 180)]:
    t0 = time.time()
    p = bvgen.make_plan("c2", n=n, bc=bc, m=m)
    tp = time.time() - t0
    bv = bvl.BlockVecchia(p)
    for _ in range(3):
        bv.loglik(theta)
    ks = []
    t = time.perf_counter()
    for _ in range(20):
        ll = bv.loglik(theta); ks.append(bv.last_kernel_ms())
    w = (time.perf_counter() - t) / 20
    print(f"bc={bc} m={m}: kernel {np.median(ks):.3f} ms, wall {w*1e3:.3f} ms, loglik {ll:.6f}, plan {tp:.1f}s", flush=True)
    bv.close()
