"""Per-phase cycle breakdown of the v3 block kernel (debug build libbv_prof.so)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bvgen  # noqa: E402
import paper_2410_04477_b200 as bvl  # noqa: E402

NAMES = ["chain: factor", "chain: wait E + arrive G", "(unused)", "chain: row solve", "chain: wait H + F + final",
         "upd: generation", "upd: GEMM + P", "upd: wait G + arrive H", "upd: row solves", "upd: U barrier",
         "upd: wait F", "upd: final + E"]


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    plan = bvgen.cached_plan(cfg)
    bv = bvl.BlockVecchia(plan)
    L = bvl.lib()
    L.bv_debug_v3_cycles.argtypes = [C.c_void_p, C.c_int]
    theta = bvgen.CONFIGS[cfg]["theta"]
    bv.loglik(theta)
    buf = (C.c_ulonglong * 16)()
    L.bv_debug_v3_cycles(buf, 1)
    bv.loglik(theta)
    L.bv_debug_v3_cycles(buf, 0)
    ctas = buf[12]
    print(f"{cfg}: kernel ms {bv.last_kernel_ms():.3f}, CTAs {ctas}")
    for i, nm in enumerate(NAMES):
        w = 1 if i < 5 else 3
        print(f"  {nm:28s} {buf[i] / ctas / w:12.0f} cycles per CTA per warp")


if __name__ == "__main__":
    main()
