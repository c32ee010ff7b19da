"""Seeded synthetic inputs for the block-Vecchia hot path (shared by both sides).

This module holds none of the likelihood's arithmetic (no covariance
function, no factorisation).  It produces:

* a counter-based RNG — SplitMix64 keyed by (seed, index), uniforms from the
  top 53 bits, normals by Box–Muller on consecutive pairs;
* the locations of the five BASELINE.json configurations (c1..c5);
* the plan — K-means blocks, random block order ζ, block nearest neighbours —
  via ``planner.cpp`` (the paper's preprocessing, Alg. 1 l.4-9,
  PAPER.md:586-591, which the paper excludes from timing);
* i.i.d. normal draws ε (the simulation noise the oracle's simulator consumes,
  and the bench's observation vector; DESIGN.md §4 explains why the bench's y
  need not be GP-distributed).

Seeds: s = 100·cfg + {1: locations, 2: y / ε, 3: K-means init, 4: ζ}.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "planner.cpp")
_LIB = os.path.join(_HERE, "_build", "libplanner.so")
_lock = threading.Lock()
_lib = None

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


# --------------------------------------------------------------------------- RNG
def _mix(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def splitmix64(seed: int, index) -> np.ndarray:
    """u64 stream value at (seed, index): mix(mix(seed + γ) + (index+1)·γ)."""
    with np.errstate(over="ignore"):
        key = _mix(np.uint64(seed) + GOLDEN)
        idx = np.asarray(index, dtype=np.uint64)
        return _mix(key + (idx + np.uint64(1)) * GOLDEN)


def uniform(seed: int, count: int, offset: int = 0) -> np.ndarray:
    """U[0,1) doubles: top 53 bits · 2⁻⁵³."""
    z = splitmix64(seed, np.arange(offset, offset + count, dtype=np.uint64))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def normal(seed: int, count: int) -> np.ndarray:
    """Standard normals by Box–Muller on consecutive uniform pairs."""
    pairs = (count + 1) // 2
    u = uniform(seed, 2 * pairs).reshape(pairs, 2)
    r = np.sqrt(-2.0 * np.log1p(-u[:, 0]))
    a = 2.0 * np.pi * u[:, 1]
    out = np.empty((pairs, 2))
    out[:, 0] = r * np.cos(a)
    out[:, 1] = r * np.sin(a)
    return out.ravel()[:count].copy()


def permutation(seed: int, count: int) -> np.ndarray:
    """Seeded Fisher–Yates (the random ordering ζ)."""
    perm = np.arange(count, dtype=np.int32)
    if count <= 1:
        return perm
    u = uniform(seed, count - 1)
    for i in range(count - 1, 0, -1):
        j = int(u[count - 1 - i] * (i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    return perm


def sample_without_replacement(seed: int, n: int, k: int) -> np.ndarray:
    """First k of a seeded partial Fisher–Yates over range(n)."""
    u = uniform(seed, k)
    pool = {}
    out = np.empty(k, dtype=np.int32)
    for i in range(k):
        j = i + int(u[i] * (n - i))
        vi, vj = pool.get(i, i), pool.get(j, j)
        out[i] = vj
        pool[j] = vi
    return out


# ---------------------------------------------------------------- planner (C++)
def build(force: bool = False) -> str:
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
                           "-o", tmp, _SRC])
    os.replace(tmp, _LIB)
    return _LIB


def _planner():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            d = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
            i32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
            i64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
            L.pl_kmeans.restype = C.c_int
            L.pl_kmeans.argtypes = [C.c_int64, C.c_int, d, C.c_int32, i32, C.c_int, i32, d, C.c_int]
            L.pl_block_nn.restype = C.c_int
            L.pl_block_nn.argtypes = [C.c_int64, C.c_int, d, C.c_int32, i32, i32, C.c_int32, i64, i32, C.c_int]
            _lib = L
    return _lib


def kmeans(locs: np.ndarray, bc: int, seed: int, max_iter: int = 100, nthreads: int = 0):
    """Lloyd K-means from a seeded uniform sample of bc points."""
    locs = np.ascontiguousarray(locs, dtype=np.float64)
    n, d = locs.shape
    init = sample_without_replacement(seed, n, bc)
    assign = np.zeros(n, dtype=np.int32)
    cent = np.zeros((bc, d))
    iters = _planner().pl_kmeans(n, d, locs, bc, init, int(max_iter), assign, cent, int(nthreads))
    return assign, cent, iters


def block_nn(locs, block_id, order, m: int, nthreads: int = 0):
    """Alg. 1 l.7-9: per position, the m nearest earlier points to the centroid."""
    locs = np.ascontiguousarray(locs, dtype=np.float64)
    n, d = locs.shape
    bc = len(order)
    ptr = np.zeros(bc + 1, dtype=np.int64)
    idx = np.zeros(max(1, bc * int(m)), dtype=np.int32)
    _planner().pl_block_nn(n, d, locs, bc, np.ascontiguousarray(block_id, dtype=np.int32),
                           np.ascontiguousarray(order, dtype=np.int32), int(m), ptr, idx, int(nthreads))
    return ptr, idx[: ptr[-1]].copy()


# ------------------------------------------------------------------- the plan
@dataclasses.dataclass
class Plan:
    """A frozen block-Vecchia plan (the bv_setup input, include/bv.h)."""
    locs: np.ndarray       # (n, d) f64, row-major
    y: np.ndarray          # (n,) f64
    block_id: np.ndarray   # (n,) i32 in [0, bc)
    order: np.ndarray      # (bc,) i32: order[k] = block at permuted position k (ζ)
    nbr_ptr: np.ndarray    # (bc+1,) i64 CSR by position
    nbr_idx: np.ndarray    # (nnz,) i32 global point ids
    name: str = ""
    m: int = 0

    @property
    def n(self):
        return int(self.locs.shape[0])

    @property
    def d(self):
        return int(self.locs.shape[1])

    @property
    def bc(self):
        return int(self.order.shape[0])

    def block_sizes(self):
        """(l_k, m_k) per permuted position k."""
        cnt = np.bincount(self.block_id, minlength=self.bc)
        return cnt[self.order].astype(np.int64), np.diff(self.nbr_ptr)

    def with_y(self, y):
        return dataclasses.replace(self, y=np.ascontiguousarray(y, dtype=np.float64))


# BASELINE.json configs (SURVEY §0 table, §8d recipe)
CONFIGS = {
    "c1": dict(cfg=1, n=2_000, d=2, bc=20, m=30, theta=(1.0, 0.078809, 0.5)),
    "c2": dict(cfg=2, n=20_000, d=2, bc=500, m=60, theta=(1.0, 0.052537, 1.5)),
    "c3": dict(cfg=3, n=250_000, d=2, bc=10_000, m=120, theta=(1.0, 0.014290, 2.5)),
    "c4": dict(cfg=4, n=1_000_000, d=3, bc=50_000, m=100, theta=(1.0, 0.052537, 1.5)),
    "c5": dict(cfg=5, n=2_000_000, d=2, bc=100_000, m=60, theta=(1.0, 0.078809, 0.5)),
}


def locations(cfg: int, n: int, d: int) -> np.ndarray:
    """c1-c3, c5: i.i.d. U[0,1]²; c4: x, y ~ U[0,1], z = k/16 with k ~ U{0..16}
    (17 layers scaled to [0,1]³; reading G16)."""
    u = uniform(100 * cfg + 1, n * d).reshape(n, d)
    if d == 3:
        u[:, 2] = np.floor(u[:, 2] * 17.0) / 16.0
    return np.ascontiguousarray(u)


def make_plan(name: str = "c1", n=None, bc=None, m=None, d=None, cfg=None, kmeans_iter=None, nthreads: int = 0,
              y: str = "normal") -> Plan:
    """Build a plan for a BASELINE config, optionally overriding sizes.

    y="normal": y = ε (i.i.d. N(0,1), seed s+2) — tests replace it with a
    GP-distributed draw from the oracle's simulator; y="zero": y = 0.
    """
    c = dict(CONFIGS[name]) if name in CONFIGS else dict(CONFIGS["c1"])
    cfg = c["cfg"] if cfg is None else cfg
    n = c["n"] if n is None else int(n)
    d = c["d"] if d is None else int(d)
    bc = c["bc"] if bc is None else int(bc)
    m = c["m"] if m is None else int(m)
    if kmeans_iter is None:
        kmeans_iter = 100 if n <= 20_000 else 20
    locs = locations(cfg, n, d)
    block_id, _, _ = kmeans(locs, bc, 100 * cfg + 3, kmeans_iter, nthreads)
    order = permutation(100 * cfg + 4, bc)
    ptr, idx = block_nn(locs, block_id, order, m, nthreads)
    yv = normal(100 * cfg + 2, n) if y == "normal" else np.zeros(n)
    return Plan(locs, yv, block_id, order, ptr, idx, name=f"{name}:n={n},bc={bc},m={m}", m=m)


def cached_plan(name: str, m=None, cache_dir=None, **kw) -> Plan:
    """make_plan with an .npz cache under <repo>/.cache/plans (not tracked)."""
    cache_dir = cache_dir or os.path.join(os.path.dirname(_HERE), ".cache", "plans")
    os.makedirs(cache_dir, exist_ok=True)
    key = name + (f"_m{m}" if m is not None else "") + "".join(f"_{k}{v}" for k, v in sorted(kw.items()))
    path = os.path.join(cache_dir, key + ".npz")
    if os.path.exists(path):
        z = np.load(path)
        return Plan(z["locs"], z["y"], z["block_id"], z["order"], z["nbr_ptr"], z["nbr_idx"], name=str(z["name"]),
                    m=int(z["m"]))
    p = make_plan(name, m=m, **kw)
    tmp = path + f".tmp{os.getpid()}.npz"
    np.savez(tmp, locs=p.locs, y=p.y, block_id=p.block_id, order=p.order, nbr_ptr=p.nbr_ptr, nbr_idx=p.nbr_idx,
             name=p.name, m=p.m)
    os.replace(tmp, path)
    return p


# --------------------------------------------------------- prediction plans (Alg. 2)
@dataclasses.dataclass
class PredPlan:
    """Inputs of Alg. 2 for n_new new locations: the clustering g of
    l.4 (block_id) and the NN sets of l.6 (CSR by prediction block; training ids)."""
    locs_new: np.ndarray
    block_id: np.ndarray
    nbr_ptr: np.ndarray
    nbr_idx: np.ndarray
    m: int = 0

    @property
    def n_new(self):
        return int(self.locs_new.shape[0])

    @property
    def bc_new(self):
        return int(self.nbr_ptr.shape[0] - 1)


def pred_nn(train_locs, centroids, m: int) -> tuple[np.ndarray, np.ndarray]:
    """Per prediction-block centroid, the m nearest TRAINING points ("m nearest
    neighbor observations from y"), ascending (squared distance summed in x, y, z order, id).
    Candidates come from a k-d tree query with 16 spare slots, then an exact re-sort."""
    from scipy.spatial import cKDTree
    train_locs = np.ascontiguousarray(train_locs, dtype=np.float64)
    n = train_locs.shape[0]
    m = int(min(m, n))
    bc = centroids.shape[0]
    ptr = np.arange(bc + 1, dtype=np.int64) * m
    if m == 0:
        return ptr, np.zeros(0, dtype=np.int32)
    k = min(n, m + 16)
    _, cand = cKDTree(train_locs).query(centroids, k=k)
    cand = np.asarray(cand).reshape(bc, k)
    idx = np.zeros(bc * m, dtype=np.int32)
    for b in range(bc):
        c = cand[b]
        diff = train_locs[c] - centroids[b]
        d2 = diff[:, 0] * diff[:, 0]
        for j in range(1, diff.shape[1]):
            d2 = d2 + diff[:, j] * diff[:, j]
        o = np.lexsort((c, d2))[:m]
        idx[b * m:(b + 1) * m] = c[o]
    return ptr, idx


def make_pred_plan(train_locs, locs_new, bc_new: int, m: int, seed: int = 9003, kmeans_iter: int = 20) -> PredPlan:
    """Alg. 2 l.4-6: K-means of the new locations into bc_new blocks, then m training NN per block
    centroid (block mean of its points)."""
    locs_new = np.ascontiguousarray(locs_new, dtype=np.float64)
    bid, cent, _ = kmeans(locs_new, int(bc_new), seed, kmeans_iter)
    ptr, idx = pred_nn(train_locs, cent, m)
    return PredPlan(locs_new, bid.astype(np.int32), ptr, idx, int(m))
