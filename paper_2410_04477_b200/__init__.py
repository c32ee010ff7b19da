"""B200-native block-Vecchia log-likelihood (arXiv 2410.04477) — Python binding.

Thin ctypes marshalling over the C ABI in ``include/bv.h`` (libbv.so, built
in-tree for sm_100a by ``paper_2410_04477_b200/build.py``).  Every step of the
evaluation runs in the library's CUDA kernels; there is no CPU fallback: if
the library or a CUDA device is missing, the calls raise.

    from paper_2410_04477_b200 import BlockVecchia
    bv = BlockVecchia(plan)                  # bv_setup
    ll = bv.loglik((1.0, 0.05, 1.5))         # bv_loglik
    ll, d, u = bv.loglik_terms(theta)        # bv_loglik_terms
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

__all__ = ["BlockVecchia", "BVError", "gpu_kmeans", "gpu_block_nn", "NotPositiveDefinite", "lib", "nccl_unique_id", "partition",
           "fixed_encode", "fixed_decode", "LIB_PATH"]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BV_LIB_PATH") or os.path.join(HERE, "libbv.so")  # override: debug builds only

BV_OK, BV_EINVAL, BV_ENOTPD, BV_EIO, BV_ECUDA, BV_ENCCL, BV_ENOMEM = 0, 2, 3, 4, 5, 6, 7
_NAMES = {2: "BV_EINVAL", 3: "BV_ENOTPD", 4: "BV_EIO", 5: "BV_ECUDA", 6: "BV_ENCCL", 7: "BV_ENOMEM"}

# every symbol include/bv.h declares (tests check the library exports them all)
EXPORTS = ["bv_version", "bv_nccl_unique_id", "bv_setup", "bv_loglik", "bv_loglik_terms", "bv_owned_range",
           "bv_loglik_host_y", "bv_last_error", "bv_launches_per_eval", "bv_stream", "bv_last_kernel_ms", "bv_destroy", "bv_partition",
           "bv_fixed_encode", "bv_fixed_decode", "bv_predict", "bv_plan_kmeans", "bv_plan_block_nn",
           "bv_plan_last_error", "bv_set_jitter", "bv_jitter_events", "bv_setup_rank_local", "bv_loglik_acc"]


class BVError(RuntimeError):
    def __init__(self, status, msg="", failed_position=-1):
        super().__init__(f"{_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.failed_position = failed_position


class NotPositiveDefinite(BVError):
    pass


class _Plan(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int32), ("locs", C.c_void_p), ("y", C.c_void_p), ("bc", C.c_int32),
                ("block_id", C.c_void_p), ("order", C.c_void_p), ("nbr_ptr", C.c_void_p), ("nbr_idx", C.c_void_p)]


class _PredPlan(C.Structure):
    _fields_ = [("n_new", C.c_int64), ("locs_new", C.c_void_p), ("bc_new", C.c_int32), ("block_id", C.c_void_p),
                ("nbr_ptr", C.c_void_p), ("nbr_idx", C.c_void_p)]


class _Dist(C.Structure):
    _fields_ = [("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("nccl_id", C.c_void_p)]


_lock = threading.Lock()
_lib = None


def lib():
    """Load libbv.so (raises if it has not been built — no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise BVError(BV_EIO, f"{LIB_PATH} not built; run python paper_2410_04477_b200/build.py")
            L = C.CDLL(LIB_PATH)
            L.bv_version.restype = C.c_char_p
            L.bv_nccl_unique_id.argtypes = [C.c_void_p]
            L.bv_setup.argtypes = [C.POINTER(_Plan), C.POINTER(_Dist), C.POINTER(C.c_void_p)]
            L.bv_setup_rank_local.argtypes = [C.POINTER(_Plan), C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
            L.bv_loglik_acc.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
            L.bv_loglik.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]
            L.bv_loglik_terms.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_double), C.c_void_p, C.c_void_p]
            L.bv_loglik_host_y.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]
            L.bv_set_jitter.argtypes = [C.c_void_p, C.c_int32]
            L.bv_jitter_events.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
            L.bv_owned_range.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
            L.bv_last_error.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_char_p)]
            L.bv_launches_per_eval.restype = C.c_int32
            L.bv_launches_per_eval.argtypes = [C.c_void_p]
            L.bv_stream.restype = C.c_void_p
            L.bv_stream.argtypes = [C.c_void_p]
            L.bv_last_kernel_ms.restype = C.c_int
            L.bv_last_kernel_ms.argtypes = [C.c_void_p, C.POINTER(C.c_float)]
            L.bv_destroy.restype = None
            L.bv_destroy.argtypes = [C.c_void_p]
            L.bv_partition.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
            L.bv_fixed_encode.argtypes = [C.c_double, C.c_void_p]
            L.bv_fixed_decode.restype = C.c_double
            L.bv_fixed_decode.argtypes = [C.c_void_p]
            L.bv_predict.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_PredPlan), C.c_void_p, C.c_void_p,
                                     C.c_void_p]
            L.bv_plan_kmeans.argtypes = [C.c_int32, C.c_int64, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                         C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)]
            L.bv_plan_block_nn.argtypes = [C.c_int32, C.c_int64, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                           C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
            L.bv_plan_last_error.restype = C.c_char_p
            for fn in ("bv_plan_kmeans", "bv_plan_block_nn", "bv_predict", "bv_nccl_unique_id", "bv_setup", "bv_loglik", "bv_loglik_terms", "bv_loglik_host_y",
                       "bv_owned_range", "bv_last_error", "bv_partition", "bv_fixed_encode", "bv_set_jitter",
                       "bv_jitter_events", "bv_setup_rank_local", "bv_loglik_acc"):
                getattr(L, fn).restype = C.c_int
            _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data if a is not None and a.size else None


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    st = lib().bv_nccl_unique_id(buf)
    if st:
        raise BVError(st, "ncclGetUniqueId failed")
    return bytes(buf)


def partition(l, m, world: int) -> np.ndarray:
    """bv_partition: contiguous cost-balanced cuts (world+1 entries)."""
    l = np.ascontiguousarray(l, dtype=np.int32)
    m = np.ascontiguousarray(m, dtype=np.int32)
    cuts = np.zeros(world + 1, dtype=np.int32)
    st = lib().bv_partition(len(l), _ptr(l), _ptr(m), int(world), cuts.ctypes.data)
    if st:
        raise BVError(st, "bv_partition")
    return cuts


def fixed_encode(t: float) -> np.ndarray:
    c = np.zeros(6, dtype=np.uint32)
    st = lib().bv_fixed_encode(float(t), c.ctypes.data)
    if st:
        raise BVError(st, "term out of fixed-point range")
    return c


def fixed_decode(acc) -> float:
    a = np.ascontiguousarray(acc, dtype=np.uint64)
    return lib().bv_fixed_decode(a.ctypes.data)


def _plan_check(st):
    if st != BV_OK:
        raise BVError(st, (lib().bv_plan_last_error() or b"").decode())


def gpu_kmeans(locs, bc: int, init_idx, max_iter: int = 100, device: int = 0):
    """Lloyd K-means on the GPU (bv_plan_kmeans; Alg. 1 l.5) →
    (assign, centroids, iterations); bit-identical to the CPU planner for the same init_idx."""
    L = lib()
    locs = np.ascontiguousarray(locs, dtype=np.float64)
    n, d = locs.shape
    init = np.ascontiguousarray(init_idx, dtype=np.int32)
    assign = np.zeros(n, dtype=np.int32)
    cent = np.zeros((bc, d))
    it = C.c_int32(0)
    _plan_check(L.bv_plan_kmeans(device, n, d, _ptr(locs), int(bc), _ptr(init), int(max_iter), _ptr(assign),
                                 _ptr(cent), C.byref(it)))
    return assign, cent, it.value


def gpu_block_nn(locs, block_id, order, m: int, device: int = 0):
    """mNearestNeighborsForBlock on the GPU (bv_plan_block_nn; Alg. 1 l.7-9) → (nbr_ptr, nbr_idx)."""
    L = lib()
    locs = np.ascontiguousarray(locs, dtype=np.float64)
    n, d = locs.shape
    bid = np.ascontiguousarray(block_id, dtype=np.int32)
    order = np.ascontiguousarray(order, dtype=np.int32)
    bc = order.shape[0]
    ptr = np.zeros(bc + 1, dtype=np.int64)
    idx = np.zeros(max(1, bc * int(m)), dtype=np.int32)
    _plan_check(L.bv_plan_block_nn(device, n, d, _ptr(locs), bc, _ptr(bid), _ptr(order), int(m), _ptr(ptr),
                                   _ptr(idx)))
    return ptr, idx[: ptr[-1]].copy()


class BlockVecchia:
    """One bv_handle: a frozen plan resident on one GPU (or one rank's share).

    ``plan`` needs numpy-convertible attributes ``locs (n,d) f64, y (n,) f64,
    block_id (n,) i32, order (bc,) i32, nbr_ptr (bc+1,) i64, nbr_idx i32``.
    For world > 1 pass rank/world and the same 128-byte ``nccl_id`` on every
    rank (see :func:`nccl_unique_id`).  ``rank_local=True`` (tests only) builds
    rank ``rank`` of ``world`` without a communicator (bv_setup_rank_local): its
    evaluations return that rank's partial sum.
    """

    def __init__(self, plan, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 rank_local: bool = False):
        L = lib()
        self._L = L
        self._h = C.c_void_p()
        locs = np.ascontiguousarray(plan.locs, dtype=np.float64)
        self._keep = dict(locs=locs, y=np.ascontiguousarray(plan.y, dtype=np.float64),
                          block_id=np.ascontiguousarray(plan.block_id, dtype=np.int32),
                          order=np.ascontiguousarray(plan.order, dtype=np.int32),
                          nbr_ptr=np.ascontiguousarray(plan.nbr_ptr, dtype=np.int64),
                          nbr_idx=np.ascontiguousarray(plan.nbr_idx, dtype=np.int32))
        k = self._keep
        self.n, self.d = locs.shape
        self.bc = int(k["order"].shape[0])
        p = _Plan(self.n, self.d, _ptr(k["locs"]), _ptr(k["y"]), self.bc, _ptr(k["block_id"]), _ptr(k["order"]),
                  _ptr(k["nbr_ptr"]), _ptr(k["nbr_idx"]))
        idbuf = None
        if world > 1 and not rank_local:
            if nccl_id is None or len(nccl_id) != 128:
                raise BVError(BV_EINVAL, "world > 1 needs a 128-byte nccl_id")
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        dist = _Dist(int(device), int(rank), int(world), C.cast(idbuf, C.c_void_p) if idbuf is not None else None)
        if rank_local:
            st = L.bv_setup_rank_local(C.byref(p), int(device), int(rank), int(world), C.byref(self._h))
        else:
            st = L.bv_setup(C.byref(p), C.byref(dist), C.byref(self._h))
        self._keep = None  # bv_setup copied everything
        if st:
            msg = C.c_char_p()
            L.bv_last_error(None, None, C.byref(msg))
            raise BVError(st, (msg.value or b"").decode())
        kb, ke = C.c_int32(), C.c_int32()
        L.bv_owned_range(self._h, C.byref(kb), C.byref(ke))
        self.k_begin, self.k_end = kb.value, ke.value

    @property
    def launches_per_eval(self) -> int:
        """Kernels per evaluation for the Matérn kind of the latest evaluation."""
        return int(self._L.bv_launches_per_eval(self._h))

    def _check(self, st):
        if st == BV_OK:
            return
        fp, msg = C.c_int32(-1), C.c_char_p()
        self._L.bv_last_error(self._h, C.byref(fp), C.byref(msg))
        cls = NotPositiveDefinite if st == BV_ENOTPD else BVError
        raise cls(st, (msg.value or b"").decode(), fp.value)

    @staticmethod
    def _theta(theta):
        return np.ascontiguousarray(theta, dtype=np.float64).reshape(3)

    def loglik(self, theta) -> float:
        """ℓ(θ) (bv_loglik).  Raises NotPositiveDefinite / BVError."""
        th = self._theta(theta)
        out = C.c_double()
        self._check(self._L.bv_loglik(self._h, th.ctypes.data, C.byref(out)))
        return out.value

    def loglik_terms(self, theta):
        """(ℓ, d_k, u_k) with d, u over this rank's positions [k_begin, k_end)."""
        th = self._theta(theta)
        nq = self.k_end - self.k_begin
        d = np.zeros(nq)
        u = np.zeros(nq)
        out = C.c_double()
        self._check(self._L.bv_loglik_terms(self._h, th.ctypes.data, C.byref(out), _ptr(d), _ptr(u)))
        return out.value, d, u

    def loglik_acc(self, theta) -> np.ndarray:
        """The evaluation's exact fixed-point accumulator (bv_loglik_acc): uint64[8] = six chunk
        sums, failed-block count, (smallest failing global position << 8 | status).  A non-PD
        evaluation still returns the accumulator."""
        th = self._theta(theta)
        acc = np.zeros(8, dtype=np.uint64)
        st = self._L.bv_loglik_acc(self._h, th.ctypes.data, acc.ctypes.data)
        if st not in (BV_OK, BV_ENOTPD):
            self._check(st)
        return acc

    def set_jitter(self, enable: bool = True):
        """Optional jitter retry for non-PD blocks (bv_set_jitter; reading G15b)."""
        self._check(self._L.bv_set_jitter(self._h, 1 if enable else 0))

    @property
    def jitter_events(self) -> int:
        """Blocks that needed jitter in the last evaluation (bv_jitter_events)."""
        ev = C.c_int64()
        self._check(self._L.bv_jitter_events(self._h, C.byref(ev)))
        return ev.value

    def loglik_host_y(self, y, theta) -> float:
        """End-to-end call: host y (global id order) copied in, ℓ back."""
        th = self._theta(theta)
        if hasattr(y, "data_ptr"):  # torch (pinned) CPU tensor: passed by pointer, so check it here
            import torch
            if y.dtype != torch.float64 or y.device.type != "cpu" or not y.is_contiguous() or y.numel() != self.n:
                raise BVError(BV_EINVAL, f"y must be a contiguous CPU float64 tensor of {self.n} elements")
            yp = y.data_ptr()
        else:
            y = np.ascontiguousarray(y, dtype=np.float64)
            if y.size != self.n:
                raise BVError(BV_EINVAL, f"y must have {self.n} elements, got {y.size}")
            yp = y.ctypes.data
        out = C.c_double()
        self._check(self._L.bv_loglik_host_y(self._h, yp, th.ctypes.data, C.byref(out)))
        return out.value

    def predict(self, theta, pred, want_cov: bool = False):
        """Alg. 2 (bv_predict): ``pred`` has locs_new (n_new,d), block_id (n_new,) i32, nbr_ptr
        (bc_new+1,) i64, nbr_idx (training ids) i32.  Returns (mean, var) or (mean, var, cov) with cov
        the blocks' l_b×l_b Σ_B* row-major, concatenated in block-id order."""
        th = self._theta(theta)
        ln = np.ascontiguousarray(pred.locs_new, dtype=np.float64)
        bid = np.ascontiguousarray(pred.block_id, dtype=np.int32)
        ptr = np.ascontiguousarray(pred.nbr_ptr, dtype=np.int64)
        idx = np.ascontiguousarray(pred.nbr_idx, dtype=np.int32)
        nn, bc = ln.shape[0], ptr.shape[0] - 1
        mean, var = np.zeros(nn), np.zeros(nn)
        cov = None
        if want_cov:
            lsz = np.bincount(bid, minlength=bc).astype(np.int64)
            cov = np.zeros(max(1, int(np.sum(lsz * lsz))))
        pp = _PredPlan(nn, _ptr(ln), bc, _ptr(bid), _ptr(ptr), idx.ctypes.data if idx.size else None)
        self._check(self._L.bv_predict(self._h, th.ctypes.data, C.byref(pp), _ptr(mean), _ptr(var),
                                       _ptr(cov) if cov is not None else None))
        return (mean, var, cov) if want_cov else (mean, var)

    @property
    def stream_ptr(self) -> int:
        """The library's cudaStream_t (for torch.cuda.ExternalStream timing)."""
        return self._L.bv_stream(self._h) or 0

    def last_kernel_ms(self) -> float:
        ms = C.c_float()
        self._check(self._L.bv_last_kernel_ms(self._h, C.byref(ms)))
        return ms.value

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.bv_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
