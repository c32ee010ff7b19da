"""Per-phase cycle breakdown of the block kernel (debug build libbv_prof.so).

    python paper_2410_04477_b200/build.py --profile-phases
    BV_LIB_PATH=paper_2410_04477_b200/libbv_prof.so python tools/phase_prof.py c4
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bvgen  # noqa: E402
import paper_2410_04477_b200 as bvl  # noqa: E402

NAMES = ["prologue+panel0", "A diag warp", "A update warps", "sync after A", "B trsm", "sync after B",
         "C + sync", "CTAs", "A upd: GEMM", "A upd: generation"]


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    plan = bvgen.cached_plan(cfg)
    bv = bvl.BlockVecchia(plan)
    L = bvl.lib()
    L.bv_debug_phase_cycles.argtypes = [C.c_void_p, C.c_int]
    theta = bvgen.CONFIGS[cfg]["theta"]
    bv.loglik(theta)
    buf = (C.c_ulonglong * 10)()
    L.bv_debug_phase_cycles(buf, 1)
    bv.loglik(theta)
    L.bv_debug_phase_cycles(buf, 0)
    ctas = buf[7]
    import re
    src = open(os.path.join(ROOT, "paper_2410_04477_b200", "csrc", "bv_block_v2.cu")).read()
    kw = int(re.search(r"constexpr int kW = (\d+);", src).group(1))
    warps_per_cta = {1: 1, 2: kw - 1, 8: kw - 1, 9: kw - 1}
    for i in (0, 3, 4, 5, 6):
        warps_per_cta[i] = kw
    print(f"{cfg}: kernel ms {bv.last_kernel_ms():.3f}, CTAs {ctas}")
    for i in (0, 1, 2, 8, 9, 3, 4, 5, 6):
        # sums are over warps (lane 0 of each warp); report per CTA per warp-role
        w = warps_per_cta.get(i, kw)
        print(f"  {NAMES[i]:18s} {buf[i] / ctas / w:12.0f} cycles per CTA (avg over {w} warps)")


if __name__ == "__main__":
    main()
