"""CPU oracle for the block-Vecchia log-likelihood (arXiv 2410.04477).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()``,
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs and the offline
diagnostics under ``tools/`` (parity_diag, pivot_floor_audit, accuracy_c5) may
import this package.  It shares no code with the CUDA product path
(``paper_2410_04477_b200``) and never imports it.

The arithmetic lives in ``bv_oracle.cpp`` (plain C++17 loops, FP64 and x87
long double, ``-ffp-contract=off``); this module only builds it and marshals
numpy arrays.  Every function cites the PAPER.md passage it follows; see the
C++ file header for the full list.

Parity status: every function here is pinned by a ``-m "not
gpu"`` test in ``tests/test_oracle_pins.py`` except the absolute value of ℓ on
large synthetic plans, which nothing outside the oracle fixes (SURVEY §8c
"parity unpinned beyond the oracle itself").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bv_oracle.cpp")
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lock = threading.Lock()
_lib = None

BV_OK, BV_EINVAL, BV_ENOTPD = 0, 2, 3

_d = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile bv_oracle.cpp → _build/liboracle.so (g++ -O2 -ffp-contract=off -fopenmp)."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(_SRC)):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
           "-shared", "-fPIC", "-o", tmp, _SRC]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            L.or_matern.restype = C.c_double
            L.or_matern.argtypes = [C.c_double] * 4 + [C.c_int]
            L.or_ln_2pi.restype = C.c_double
            L.or_ln_2pi.argtypes = [C.c_int]
            L.or_potrf.restype = C.c_int
            L.or_potrf.argtypes = [_d, C.c_int, _d]
            L.or_trsv.restype = None
            L.or_trsv.argtypes = [_d, C.c_int, _d]
            L.or_bv_loglik.restype = C.c_int
            L.or_bv_loglik.argtypes = [C.c_int64, C.c_int, _d, _d, C.c_int32, _i32, _i32, _i64, _i32, _d,
                                       C.c_int, C.c_int, C.c_int32, C.c_int32,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_double),
                                       C.POINTER(C.c_int32), C.c_uint32]
            L.or_bv_loglik_joint.restype = C.c_int
            L.or_bv_loglik_joint.argtypes = [C.c_int64, C.c_int, _d, _d, C.c_int32, _i32, _i32, _i64, _i32, _d,
                                             C.c_int, C.c_int, C.c_int32, C.c_int32,
                                             C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_double),
                                             C.POINTER(C.c_int32)]
            L.or_bv_loglik_jitter.restype = C.c_int
            L.or_bv_loglik_jitter.argtypes = [C.c_int64, C.c_int, _d, _d, C.c_int32, _i32, _i32, _i64, _i32, _d,
                                              C.c_int, C.c_int32, C.c_int32, _d, _d, _d, _d,
                                              C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
            L.or_exact_loglik.restype = C.c_int
            L.or_exact_loglik.argtypes = [C.c_int64, C.c_int, _d, _d, _d, C.c_int, C.POINTER(C.c_double)]
            L.or_classic_vecchia.restype = C.c_int
            L.or_classic_vecchia.argtypes = [C.c_int64, C.c_int, _d, _d, _i32, _i64, _i32, _d,
                                             C.POINTER(C.c_double)]
            L.or_simulate_bv.restype = C.c_int
            L.or_simulate_bv.argtypes = [C.c_int64, C.c_int, _d, C.c_int32, _i32, _i32, _i64, _i32, _d, _d, _d,
                                         C.c_int]
            L.or_simulate_exact.restype = C.c_int
            L.or_simulate_exact.argtypes = [C.c_int64, C.c_int, _d, _d, _d, _d]
            L.or_block_nn_bruteforce.restype = C.c_int
            L.or_block_nn_bruteforce.argtypes = [C.c_int64, C.c_int, _d, C.c_int32, _i32, _i32, C.c_int32, _i64,
                                                 _i32]
            L.or_bv_predict.restype = C.c_int
            L.or_bv_predict.argtypes = [C.c_int64, C.c_int, _d, _d, _d, C.c_int64, _d, C.c_int32, _i32, _i64, _i32,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)]
            L.or_kmeans_assign_bruteforce.restype = None
            L.or_kmeans_assign_bruteforce.argtypes = [C.c_int64, C.c_int, _d, C.c_int32, _d, _i32]
            _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, status, failed_position=-1):
        super().__init__(f"oracle status {status} (failed position {failed_position})")
        self.status = status
        self.failed_position = failed_position


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def matern(r, theta, mode: int = 0):
    """Eq. (7).  mode 0 dispatching, 1 general K_ν, 2 long double."""
    L = lib()
    s2, be, nu = (float(t) for t in theta)
    r = np.asarray(r, dtype=np.float64)
    out = np.array([L.or_matern(float(x), s2, be, nu, mode) for x in r.ravel()])
    return out.reshape(r.shape)


def ln_2pi(long_double: bool = False) -> float:
    return lib().or_ln_2pi(1 if long_double else 0)


def potrf(A):
    A = _c(A, np.float64)
    n = A.shape[0]
    Lm = np.zeros_like(A)
    st = lib().or_potrf(A, n, Lm)
    if st:
        raise OracleError(st)
    return Lm


def trsv(Lm, b):
    Lm = _c(Lm, np.float64)
    x = _c(b, np.float64).copy()
    lib().or_trsv(Lm, Lm.shape[0], x)
    return x


def bv_loglik(plan, theta, long_double: bool = False, nthreads: int = 0, k_range=None, per_block: bool = True,
              perturb_seed: int = 0):
    """Alg. 1 literally.  Returns dict(loglik, u, d, t).

    ``plan`` carries numpy arrays ``locs (n,d) f64, y (n,) f64, block_id (n,)
    i32, order (bc,) i32, nbr_ptr (bc+1,) i64, nbr_idx (nnz,) i32``.
    ``k_range`` = (k_begin, k_end) restricts to those permuted positions.
    Raises OracleError(3, k) on a non-PD block (k = smallest failing position).
    ``perturb_seed`` != 0 moves every off-diagonal covariance entry by −1/0/+1
    ulp (a fixed function of the point pair and the seed): the spread over a
    few seeds estimates FP64's own error (parity reading G22).
    """
    L = lib()
    locs = _c(plan.locs, np.float64)
    n, d = locs.shape
    bc = int(plan.order.shape[0])
    kb, ke = (0, bc) if k_range is None else (int(k_range[0]), int(k_range[1]))
    nk = ke - kb
    u = np.zeros(nk) if per_block else None
    dd = np.zeros(nk) if per_block else None
    t = np.zeros(nk) if per_block else None
    ll = C.c_double(0.0)
    fp = C.c_int32(-1)
    th = _c(theta, np.float64)
    st = L.or_bv_loglik(n, d, locs, _c(plan.y, np.float64), bc, _c(plan.block_id, np.int32),
                        _c(plan.order, np.int32), _c(plan.nbr_ptr, np.int64), _c(plan.nbr_idx, np.int32), th,
                        1 if long_double else 0, int(nthreads), kb, ke,
                        u.ctypes.data if per_block else None, dd.ctypes.data if per_block else None,
                        t.ctypes.data if per_block else None, C.byref(ll), C.byref(fp), int(perturb_seed))
    if st:
        raise OracleError(st, fp.value)
    return {"loglik": ll.value, "u": u, "d": dd, "t": t}


def set_pivot_floor(f: float = 1e-14):
    """Reading G15's non-PD floor (a pivot must exceed f·σ²; 0 = plain "≤ 0"), process-global.
    For the floor audit (tools/pivot_floor_audit.py); every other caller keeps the default."""
    L = lib()
    L.or_set_pivot_floor.argtypes = [C.c_double]
    L.or_set_pivot_floor.restype = None
    L.or_set_pivot_floor(float(f))


def bv_loglik_joint(plan, theta, long_double: bool = False, nthreads: int = 0):
    """DIAGNOSTIC ONLY (not a parity reference): the block terms through the joint-Cholesky
    formulation (or_bv_loglik_joint), to measure how far two exact FP64 formulations of Alg. 1
    differ on ill-conditioned blocks (tools/parity_diag.py, reading G22)."""
    L = lib()
    locs = _c(plan.locs, np.float64)
    n, d = locs.shape
    bc = int(plan.order.shape[0])
    u, dd, t = np.zeros(bc), np.zeros(bc), np.zeros(bc)
    ll = C.c_double(0.0)
    fp = C.c_int32(-1)
    st = L.or_bv_loglik_joint(n, d, locs, _c(plan.y, np.float64), bc, _c(plan.block_id, np.int32),
                              _c(plan.order, np.int32), _c(plan.nbr_ptr, np.int64), _c(plan.nbr_idx, np.int32),
                              _c(theta, np.float64), 1 if long_double else 0, int(nthreads), 0, bc, u.ctypes.data,
                              dd.ctypes.data, t.ctypes.data, C.byref(ll), C.byref(fp))
    if st:
        raise OracleError(st, fp.value)
    return {"loglik": ll.value, "u": u, "d": dd, "t": t}


def bv_loglik_jitter(plan, theta, nthreads: int = 0):
    """Alg. 1 with the optional jitter mode (reading G15b; SPEC.md:197,
    :238 schedule with base_scale = σ²): a block whose POTRF fails is re-run with
    ε·σ² added to the diagonal of Σcon and Σlk, ε = 1e-10, 1e-8, 1e-6 in turn.
    Returns dict(loglik, u, d, t, eps (per block, 0 = none), events)."""
    L = lib()
    locs = _c(plan.locs, np.float64)
    n, d = locs.shape
    bc = int(plan.order.shape[0])
    u, dd, t, eps = (np.zeros(bc) for _ in range(4))
    ll, fp, ev = C.c_double(0.0), C.c_int32(-1), C.c_int32(0)
    st = L.or_bv_loglik_jitter(n, d, locs, _c(plan.y, np.float64), bc, _c(plan.block_id, np.int32),
                               _c(plan.order, np.int32), _c(plan.nbr_ptr, np.int64), _c(plan.nbr_idx, np.int32),
                               _c(theta, np.float64), int(nthreads), 0, bc, u, dd, t, eps, C.byref(ll),
                               C.byref(fp), C.byref(ev))
    if st:
        raise OracleError(st, fp.value)
    return {"loglik": ll.value, "u": u, "d": dd, "t": t, "eps": eps, "events": ev.value}


def exact_loglik(locs, y, theta, long_double: bool = False) -> float:
    """Eq. (1), dense Cholesky; n ≤ 6000."""
    locs = _c(locs, np.float64)
    out = C.c_double(0.0)
    st = lib().or_exact_loglik(locs.shape[0], locs.shape[1], locs, _c(y, np.float64), _c(theta, np.float64),
                               1 if long_double else 0, C.byref(out))
    if st:
        raise OracleError(st)
    return out.value


def classic_vecchia(locs, y, point_order, nbr_ptr, nbr_idx, theta) -> float:
    """Textbook classic Vecchia by Gaussian elimination."""
    locs = _c(locs, np.float64)
    out = C.c_double(0.0)
    st = lib().or_classic_vecchia(locs.shape[0], locs.shape[1], locs, _c(y, np.float64), _c(point_order, np.int32),
                                  _c(nbr_ptr, np.int64), _c(nbr_idx, np.int32), _c(theta, np.float64),
                                  C.byref(out))
    if st:
        raise OracleError(st)
    return out.value


def simulate_bv(plan, theta, eps, nthreads: int = 0):
    """Block-Vecchia sequential simulation from the plan → y."""
    locs = _c(plan.locs, np.float64)
    n, d = locs.shape
    y = np.zeros(n)
    st = lib().or_simulate_bv(n, d, locs, int(plan.order.shape[0]), _c(plan.block_id, np.int32),
                              _c(plan.order, np.int32), _c(plan.nbr_ptr, np.int64), _c(plan.nbr_idx, np.int32),
                              _c(theta, np.float64), _c(eps, np.float64), y, int(nthreads))
    if st:
        raise OracleError(st)
    return y


def simulate_exact(locs, theta, eps):
    """Exact GRF y = chol(Σθ) ε (n ≤ 6000)."""
    locs = _c(locs, np.float64)
    y = np.zeros(locs.shape[0])
    st = lib().or_simulate_exact(locs.shape[0], locs.shape[1], locs, _c(theta, np.float64), _c(eps, np.float64), y)
    if st:
        raise OracleError(st)
    return y


def block_nn_bruteforce(locs, block_id, order, m):
    """Alg. 1 l.7-9 by O(n²) brute force → (nbr_ptr, nbr_idx)."""
    locs = _c(locs, np.float64)
    n, d = locs.shape
    bc = int(len(order))
    ptr = np.zeros(bc + 1, dtype=np.int64)
    idx = np.zeros(max(1, bc * int(m)), dtype=np.int32)
    lib().or_block_nn_bruteforce(n, d, locs, bc, _c(block_id, np.int32), _c(order, np.int32), int(m), ptr, idx)
    return ptr, idx[: ptr[-1]].copy()


def kmeans_assign_bruteforce(locs, centroids):
    locs = _c(locs, np.float64)
    cent = _c(centroids, np.float64)
    out = np.zeros(locs.shape[0], dtype=np.int32)
    lib().or_kmeans_assign_bruteforce(locs.shape[0], locs.shape[1], locs, cent.shape[0], cent, out)
    return out


def bv_predict(locs, y, theta, locs_new, block_new, nbr_ptr, nbr_idx, want_cov: bool = False):
    """Alg. 2 literally → dict(mean, var[, cov (flat, per block l_b² row-major)])."""
    locs = _c(locs, np.float64)
    n, d = locs.shape
    ln = _c(locs_new, np.float64)
    bn = _c(block_new, np.int32)
    bc = int(bn.max()) + 1 if bn.size else 0
    mean = np.zeros(ln.shape[0])
    var = np.zeros(ln.shape[0])
    lsz = np.bincount(bn, minlength=bc).astype(np.int64)
    cov = np.zeros(int(np.sum(lsz * lsz))) if want_cov else None
    fb = C.c_int32(-1)
    st = lib().or_bv_predict(n, d, locs, _c(y, np.float64), _c(theta, np.float64), ln.shape[0], ln, bc, bn,
                             _c(nbr_ptr, np.int64), _c(nbr_idx, np.int32), mean.ctypes.data, var.ctypes.data,
                             cov.ctypes.data if cov is not None else None, C.byref(fb))
    if st:
        raise OracleError(st, fb.value)
    out = {"mean": mean, "var": var}
    if cov is not None:
        out["cov"] = cov
    return out
