"""Build the in-tree CUDA library libbv.so for sm_100a (nvcc, no JIT cache).

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC
Links NCCL from the torch-bundled nvidia-nccl wheel (same soname torch loads).
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbv.so")
SOURCES = ["bv_host.cpp", "bv_kernels.cu", "bv_block_v3.cu", "bv_block_w.cu", "bv_predict.cu", "bv_cv.cu", "bv_plan.cu"]
HEADERS = ["bv_common.cuh", "matern.cuh", "bessel_k.cuh", "bv_tile.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        base = list(spec.submodule_search_locations)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "bv.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, profile_phases: bool = False, variant: str = "",
          defines=()) -> str:
    """Build libbv.so (or, with profile_phases, the debug-instrumented libbv_prof.so;
    with variant="x" and defines, an experimental libbv_x.so for A/B timing)."""
    out = LIB if not profile_phases else os.path.join(HERE, "libbv_prof.so")
    if variant:
        out = os.path.join(HERE, f"libbv_{variant}.so")
    if not profile_phases and not variant and not force and not _stale():
        return LIB
    inc, libdir = nccl_dirs()
    tmp = out + f".tmp{os.getpid()}"
    extra = (["-DBV_PROFILE_PHASES"] if profile_phases else []) + [f"-D{d}" for d in defines]
    flags = [*ARCH, *extra, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc]
    # one nvcc per translation unit, in parallel (the v3 kernel's instantiations dominate), then link
    objs = [f"{tmp}.{i}.o" for i in range(len(SOURCES))]
    split = lambda f: ["-split-compile=4"] if f.startswith("bv_block_v") else []
    procs = [subprocess.Popen(["nvcc", *flags, *split(f), "-c", os.path.join(CSRC, f), "-o", o])
             for f, o in zip(SOURCES, objs)]
    rcs = [p.wait() for p in procs]
    try:
        if any(rcs):
            raise subprocess.CalledProcessError(max(rcs), "nvcc -c " + " ".join(SOURCES))
        subprocess.check_call(["nvcc", *ARCH, "-shared", "-o", tmp, *objs,
                               "-L", libdir, "-l:libnccl.so.2", f"-Xlinker=-rpath,{libdir}"])
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    os.replace(tmp, out)
    return out


def build_ablation(force: bool = False) -> str:
    """libbv_fill.so: the timing ablation of SURVEY §8d (v) — Matérn fill replaced by a cheap
    SPD fill (-DBV_ABL_FILL).  Diagnostic only; bench.py reports it as `factorization_only`."""
    out = os.path.join(HERE, "libbv_fill.so")
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(LIB):
        build(variant="fill", defines=["BV_ABL_FILL"])
    return out


if __name__ == "__main__":
    var = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")]
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                profile_phases="--profile-phases" in sys.argv, variant=var[0] if var else "", defines=defs))
