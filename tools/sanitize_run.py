"""Small evaluations that reach every block kernel, for compute-sanitizer runs (one tool per call):
    compute-sanitizer --tool {racecheck,synccheck,memcheck} python tools/sanitize_run.py
  * c1-shaped plan: CTA kernel (bv_block_v3) across several tile-row buckets, warp kernel for the
    small ones;  * bc = n, m = 20: classic-Vecchia warp kernel (bv_cv);  * joint sizes ≈ 450: the CTA
    kernel with global-memory tile slots (persistent CTAs);  * a small-block plan: warp-per-block
    kernel (bv_block_w);  * general ν on a small plan: the pre-generation kernel + KIND kPre;
  * the jitter retry (a repeated location)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bvgen  # noqa: E402
from paper_2410_04477_b200 import BlockVecchia, NotPositiveDefinite  # noqa: E402


def run(p, theta, tag):
    bv = BlockVecchia(p)
    ll = bv.loglik(theta)
    print(tag, "launches", bv.launches_per_eval, "loglik", ll, flush=True)
    bv.close()


def main():
    th = (1.0, 0.09, 1.5)
    run(bvgen.make_plan("c1", n=2000, bc=20, m=30, cfg=1), th, "c1-shaped (v3 buckets)")
    run(bvgen.make_plan("c1", n=800, bc=800, m=20, cfg=38), th, "bc=n (cv)")
    run(bvgen.make_plan("c1", n=900, bc=6, m=300, cfg=31), th, "N~450 (v3 global slots)")
    run(bvgen.make_plan("c1", n=4000, bc=200, m=30, cfg=40), th, "small blocks (warp kernel)")
    run(bvgen.make_plan("c1", n=3000, bc=60, m=30, cfg=41), (1.1, 0.06, 0.83), "general nu (pregen + kPre)")
    p = bvgen.make_plan("c1", n=400, bc=16, m=20, cfg=33)
    locs = p.locs.copy()
    mem = np.where(p.block_id == p.order[9])[0]
    locs[mem[1]] = locs[mem[0]]
    q = bvgen.Plan(locs, bvgen.normal(4401, p.n), p.block_id, p.order, p.nbr_ptr, p.nbr_idx)
    bv = BlockVecchia(q)
    try:
        bv.loglik(th)
    except NotPositiveDefinite as e:
        print("non-PD at", e.failed_position)
    bv.set_jitter(True)
    print("jitter", bv.loglik(th), bv.jitter_events)
    bv.close()


if __name__ == "__main__":
    main()
