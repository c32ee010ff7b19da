"""Minimal profiling target: set up one config and run a few evaluations.

    python tools/prof_run.py [config] [evals] [m]
Used under `ncu` (one GPU) to capture the block kernels; prints the per-bucket
launch plan so the ncu launch list can be mapped back to tile sizes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bvgen  # noqa: E402
import paper_2410_04477_b200 as bvl  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    evals = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    m = int(sys.argv[3]) if len(sys.argv) > 3 else None
    plan = bvgen.cached_plan(cfg, m=m)
    l, m = plan.block_sizes()
    TI = (l + m + 8) // 8
    vals, cnts = np.unique(TI, return_counts=True)
    print("buckets (TI: count), largest first:", dict(zip(vals[::-1].tolist(), cnts[::-1].tolist())))
    bv = bvl.BlockVecchia(plan)
    theta = bvgen.CONFIGS[cfg]["theta"]
    for i in range(evals):
        ll = bv.loglik(theta)
    print("launches/eval", bv.launches_per_eval, "loglik", ll, "kernel ms", bv.last_kernel_ms())


if __name__ == "__main__":
    main()
