"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle (-m gpu).

Same seeded inputs on both sides (bvgen plan + y drawn by the oracle's
block-Vecchia simulator at θ, so y follows the model — SURVEY §8c P11a).
Full element-wise comparison at c1, c2 and c3 sizes; at c4 (n = 1M, 3D) the
whole ℓ plus element-wise terms on sampled position ranges (the densest tail
and the head), in the launch configuration bench.py times.
"""
import math
import os

import numpy as np
import pytest

import bvgen
import oracle
from paper_2410_04477_b200 import BlockVecchia, BVError, NotPositiveDefinite
from paper_2410_04477_b200 import build as bvbuild

from parity import compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    bvbuild.build()


def sim_plan(name, theta, seed_eps=None, **kw):
    p = bvgen.cached_plan(name, **kw) if not kw or "n" not in kw else bvgen.make_plan(name, **kw)
    cfg = bvgen.CONFIGS.get(name, {"cfg": 9})["cfg"]
    eps = bvgen.normal(seed_eps if seed_eps is not None else 100 * cfg + 2, p.n)
    return p.with_y(oracle.simulate_bv(p, theta, eps))


def replicas(p, theta, k_range=None):
    """FP64 oracle runs with entries moved by up to ±2 ulp (parity reading G22): six
    equally valid FP64 evaluations of Eq. (7), whose spread sizes FP64's own error."""
    return [oracle.bv_loglik(p, theta, k_range=k_range, perturb_seed=2000 + s) for s in range(1, 7)]


def full_parity(p, theta, label):
    bv = BlockVecchia(p)
    ll, d, u = bv.loglik_terms(theta)
    o64 = oracle.bv_loglik(p, theta)
    old = oracle.bv_loglik(p, theta, long_double=True)
    l, _ = p.block_sizes()
    s = compare(d, u, o64, old, l, ll, o64["loglik"], label, replicas=replicas(p, theta))
    print(label, s)
    bv.close()
    return s


@pytest.mark.parametrize("theta", [(1.0, 0.078809, 0.5), (1.0, 0.078809, 1.5), (1.0, 0.078809, 2.5),
                                   (1.3, 0.05, 0.83), (0.8, 0.03, 1.0),
                                   (1.0, 0.004, 1.7), (1.3, 0.3, 0.35), (0.7, 0.02, 2.9)])
def test_c1_full_parity(theta):
    """Closed-form ν and general ν across all three K_ν regimes of the device evaluator
    (Temme x ≤ 2, trapezoid 2 < x ≤ 22, asymptotic x > 22: β = 0.004 puts most pairs there)."""
    p = sim_plan("c1", theta)
    full_parity(p, theta, f"c1 {theta}")


@pytest.mark.parametrize("theta", [(1.0, 0.052537, 1.5), (0.9, 0.06, 1.31)])
def test_c2_full_parity(theta):
    p = sim_plan("c2", theta)
    full_parity(p, theta, f"c2 {theta}")


@pytest.mark.parametrize("theta", [(1.0, 0.0025, 2.5), (1.0, 0.014290, 2.5)])
def test_c3_full_parity(theta):
    """c3 at the strict-graded β=0.0025 and at Table 1 β (κ-aware branch expected)."""
    p = sim_plan("c3", theta)
    full_parity(p, theta, f"c3 {theta}")


def test_c4_full_size_sampled_parity():
    """n = 1M 3D (the headline config): whole ℓ vs the FP64 oracle; terms element-wise on
    the first 500 and the densest last 2000 positions (long-double oracle there)."""
    theta = (1.0, 0.017512, 1.5)
    p = sim_plan("c4", theta)
    bv = BlockVecchia(p)
    ll, d, u = bv.loglik_terms(theta)
    o64 = oracle.bv_loglik(p, theta, per_block=True)
    rel = abs(ll - o64["loglik"]) / abs(o64["loglik"])
    assert rel <= 1e-9, rel
    l, _ = p.block_sizes()
    for a, b in ((0, 500), (p.bc - 2000, p.bc)):
        old = oracle.bv_loglik(p, theta, long_double=True, k_range=(a, b))
        sub = {k: o64[k][a:b] for k in ("u", "d", "t")}
        s = compare(d[a:b], u[a:b], sub, old, l[a:b], label=f"c4[{a}:{b}]",
                    replicas=replicas(p, theta, k_range=(a, b)))
        print("c4", a, b, s, "ll rel", rel)
    # timed theta too (bench.py's), whole ℓ only
    th2 = (1.0, 0.052537, 1.5)
    ll2 = bv.loglik(th2)
    o2 = oracle.bv_loglik(p, th2, per_block=False)["loglik"]
    assert abs(ll2 - o2) <= 1e-9 * abs(o2)
    bv.close()


def test_c5_shaped_m200_sampled_parity():
    """c5's block-size mix at m = 200 (joint sizes to ~263, beyond the 240 a packed triangle fits;
    the left-looking slot layout runs them one CTA per SM) at n = 200k: whole ℓ vs the FP64 oracle
    and element-wise terms on the largest-N positions and the head.  y is simulated once with the
    nested m = 60 plan (c5 y generated with m_sim = 60)."""
    theta = (1.0, 0.078809, 0.5)
    kw = dict(n=200_000, bc=10_000, cfg=5)
    p60 = bvgen.make_plan("c5", m=60, **kw)
    y = oracle.simulate_bv(p60, theta, bvgen.normal(502, p60.n))
    p = bvgen.make_plan("c5", m=200, **kw).with_y(y)
    l, mk = p.block_sizes()
    N = l + mk
    assert N.max() > 240
    bv = BlockVecchia(p)
    ll, d, u = bv.loglik_terms(theta)
    o64 = oracle.bv_loglik(p, theta, per_block=True)
    rel = abs(ll - o64["loglik"]) / abs(o64["loglik"])
    assert rel <= 1e-9, rel
    big = np.sort(np.argsort(-N, kind="stable")[:300])
    for idx, lab in ((big, "largest N"), (np.arange(300), "head")):
        dd, uu = d[idx], u[idx]
        od, ou = o64["d"][idx], o64["u"][idx]
        sc = np.abs(ou) + np.abs(od) + l[idx] * 1.8378770664093456
        e = max(np.max(np.abs(dd - od) / sc), np.max(np.abs(uu - ou) / sc))
        print("c5 m=200", lab, "max term err", e, "ll rel", rel)
        assert e <= 1e-10, (lab, e)  # ν = 0.5: κ ≤ 3e6, strict bar everywhere
    bv.close()


# ---------------------------------------------------------------- edge cases
@pytest.mark.parametrize("n,bc,m,d", [
    (50, 1, 10, 2),        # one block, no neighbours (m_1 = 0)
    (40, 40, 6, 2),        # singleton blocks = classic Vecchia
    (97, 13, 0, 2),        # m = 0 everywhere: independent blocks
    (333, 17, 45, 3),      # ragged 3D
    (700, 7, 100, 2),      # large blocks (N ≈ 200)
    (64, 2, 70, 2),        # second block conditions on all of the first (m > l_1)
    (600, 6, 180, 2),      # joint sizes up to ~280 (c5 at m = 200 reaches 263): one CTA per SM
    (900, 6, 300, 2),      # joint sizes ~450 (the paper's cs = 420-450): tile slots in global scratch
    (700, 7, 330, 3),      # 3D, joint sizes ~430, persistent CTAs over the global-slot bucket
])
def test_edge_shapes_parity(n, bc, m, d):
    theta = (1.2, 0.09, 1.5)
    p = bvgen.make_plan("c4" if d == 3 else "c1", n=n, bc=bc, m=m, d=d, cfg=31)
    p = p.with_y(oracle.simulate_bv(p, theta, bvgen.normal(3102, n)))
    full_parity(p, theta, f"edge n={n} bc={bc} m={m} d={d}")


def test_single_block_equals_exact_on_gpu():
    """bc = 1: the GPU ℓ equals Eq. (1) (oracle's dense exact ℓ)."""
    theta = (1.0, 0.1, 2.5)
    p = bvgen.make_plan("c1", n=120, bc=1, m=5, cfg=32)
    p = p.with_y(oracle.simulate_exact(p.locs, theta, bvgen.normal(7, p.n)))
    ll = BlockVecchia(p).loglik(theta)
    ex = oracle.exact_loglik(p.locs, p.y, theta, long_double=True)
    assert abs(ll - ex) <= 1e-10 * abs(ex)


def test_not_pd_reports_smallest_position():
    theta = (1.0, 0.1, 0.5)
    p = bvgen.make_plan("c1", n=400, bc=16, m=20, cfg=33)
    locs = p.locs.copy()
    for k in (9, 4):  # duplicate a point inside the blocks at positions 9 and 4
        mem = np.where(p.block_id == p.order[k])[0]
        locs[mem[1]] = locs[mem[0]]
    q = bvgen.Plan(locs, p.y, p.block_id, p.order, p.nbr_ptr, p.nbr_idx)
    with pytest.raises(oracle.OracleError) as eo:
        oracle.bv_loglik(q, theta)
    with pytest.raises(NotPositiveDefinite) as eg:
        BlockVecchia(q).loglik(theta)
    assert eg.value.failed_position == eo.value.failed_position
    assert eg.value.failed_position <= 4


def test_invalid_theta_rejected():
    p = bvgen.make_plan("c1", n=100, bc=5, m=5, cfg=34)
    bv = BlockVecchia(p)
    for th in [(0.0, 0.1, 0.5), (1.0, -1.0, 0.5), (1.0, 0.1, float("nan")), (float("inf"), 0.1, 0.5)]:
        with pytest.raises(BVError) as e:
            bv.loglik(th)
        assert e.value.status == 2


# ---------------------------------------------------------------- properties
def test_determinism_and_host_y_path():
    theta = (1.0, 0.052537, 1.5)
    p = sim_plan("c2", theta)
    bv = BlockVecchia(p)
    a = bv.loglik(theta)
    b = bv.loglik((2.0, 0.1, 0.5))
    c = bv.loglik(theta)
    assert a == c and a != b
    assert bv.loglik_host_y(p.y, theta) == a
    # a different y through the e2e path, then back
    y2 = p.y * 0.5
    assert bv.loglik_host_y(y2, theta) != a
    assert bv.loglik_host_y(p.y, theta) == a


def test_gpu_sigma2_and_length_scaling_exact():
    """Metamorphic pins on the GPU path: σ²×4 → u/4 bitwise;
    (coords, β)×2^k → (u, d) bitwise."""
    theta = (1.0, 0.06, 1.5)
    p = bvgen.make_plan("c1", n=3000, bc=150, m=40, cfg=35)
    p = p.with_y(oracle.simulate_bv(p, theta, bvgen.normal(3502, p.n)))
    _, d1, u1 = BlockVecchia(p).loglik_terms(theta)
    _, d4, u4 = BlockVecchia(p).loglik_terms((4.0, 0.06, 1.5))
    assert np.array_equal(u4, u1 / 4)
    l, _ = p.block_sizes()
    assert np.all(np.abs(d4 - d1 - 2 * l * math.log(2.0)) <= 1e-13 * (np.abs(d1) + l))
    q = bvgen.Plan(p.locs * 8.0, p.y, p.block_id, p.order, p.nbr_ptr, p.nbr_idx)
    _, d8, u8 = BlockVecchia(q).loglik_terms((1.0, 0.48, 1.5))
    assert np.array_equal(u8, u1) and np.array_equal(d8, d1)


def test_generating_model_on_gpu():
    """u_k = ‖ε_k‖² when y is simulated block-sequentially (construction pin, any size)."""
    theta = (1.0, 0.078809, 0.5)
    p = bvgen.make_plan("c1")
    eps = bvgen.normal(102, p.n)
    p = p.with_y(oracle.simulate_bv(p, theta, eps))
    _, d, u = BlockVecchia(p).loglik_terms(theta)
    e2 = np.array([np.sum(eps[np.where(p.block_id == b)[0]] ** 2) for b in p.order])
    assert np.max(np.abs(u - e2) / e2) <= 1e-11


def test_joint_size_beyond_limit_rejected():
    """N = m + l above the largest joint size this build supports (480: shared-memory slots to 295,
    global-memory slots to 480) → BV_EINVAL naming the first offending position, never a silent
    fallback."""
    p = bvgen.make_plan("c1", n=1200, bc=2, m=400, cfg=33)
    l, mk = p.block_sizes()
    assert (l + mk).max() > 480
    with pytest.raises(BVError) as ei:
        BlockVecchia(p, device=0)
    assert ei.value.status == 2 and "largest joint size" in str(ei.value)


# ------------------------------------------------------- classic Vecchia
@pytest.mark.parametrize("theta,m", [((1.0, 0.078809, 0.5), 30), ((1.0, 0.052537, 1.5), 20),
                                     ((0.9, 0.06, 1.31), 31), ((1.2, 0.1, 2.5), 8)])
def test_classic_vecchia_warp_kernel_parity(theta, m):
    """bc = n (block size 1) runs the warp-per-position kernel (bv_cv.cu): terms and ℓ
    vs the FP64/80-bit oracle (Alg. 1 literal), and ℓ vs the textbook classic-Vecchia oracle."""
    n = 1500
    p = bvgen.make_plan("c1", n=n, bc=n, m=m, cfg=37)
    p = p.with_y(oracle.simulate_bv(p, theta, bvgen.normal(3702, n)))
    s = full_parity(p, theta, f"cv m={m} {theta}")
    pt = np.empty(n, dtype=np.int32)  # singleton block b holds point pt[b]
    pt[p.block_id] = np.arange(n, dtype=np.int32)
    point_order = pt[p.order]
    cv = oracle.classic_vecchia(p.locs, p.y, point_order, p.nbr_ptr, p.nbr_idx, theta)
    bv = BlockVecchia(p)
    ll = bv.loglik(theta)
    bv.close()
    assert abs(ll - cv) <= 1e-9 * abs(cv), (ll, cv)


def test_classic_vecchia_kernel_equals_block_kernel(monkeypatch):
    """The same bc = n plan through the warp kernel and (BV_NO_CV=1) through the block kernel."""
    theta = (1.0, 0.078809, 1.5)
    p = bvgen.make_plan("c1", n=800, bc=800, m=25, cfg=38)
    p = p.with_y(oracle.simulate_bv(p, theta, bvgen.normal(3802, 800)))
    a = BlockVecchia(p)
    la, da, ua = a.loglik_terms(theta)
    a.close()
    monkeypatch.setenv("BV_NO_CV", "1")
    b = BlockVecchia(p)
    lb, db, ub = b.loglik_terms(theta)
    b.close()
    sc = np.abs(ua) + np.abs(da) + 1.8378770664093456
    assert np.max(np.abs(da - db) / sc) <= 1e-12 and np.max(np.abs(ua - ub) / sc) <= 1e-12
    assert abs(la - lb) <= 1e-12 * abs(la)


def _dup_plan_gpu(positions, n=400, bc=16, m=20, cfg=33):
    p = bvgen.make_plan("c1", n=n, bc=bc, m=m, cfg=cfg)
    locs = p.locs.copy()
    y = bvgen.normal(4401, p.n)
    for k in positions:  # a repeated location inside the block at position k
        mem = np.where(p.block_id == p.order[k])[0]
        locs[mem[1]] = locs[mem[0]]
        y[mem[1]] = y[mem[0]] + 1e-6
    return bvgen.Plan(locs, y, p.block_id, p.order, p.nbr_ptr, p.nbr_idx)


@pytest.mark.parametrize("theta", [(1.0, 0.1, 0.5), (1.3, 0.12, 1.5), (0.7, 0.1, 0.83)])
def test_jitter_mode_matches_oracle(theta):
    """Optional jitter mode (reading G15b): the GPU retries exactly the oracle's blocks
    with the same ε; jittered blocks agree to the conditioning the 1e-10 jitter leaves
    (κ ≈ 1e10), all others to the usual FP64 bound; ℓ and jitter_events agree."""
    q = _dup_plan_gpu((9, 4))
    o = oracle.bv_loglik_jitter(q, theta)
    assert o["events"] >= 2
    bv = BlockVecchia(q)
    with pytest.raises(NotPositiveDefinite):
        bv.loglik(theta)  # mode off by default
    assert bv.jitter_events == 0
    bv.set_jitter(True)
    ll, d, u = bv.loglik_terms(theta)
    assert bv.jitter_events == o["events"]
    l, _ = q.block_sizes()
    scale = np.abs(o["u"]) + np.abs(o["d"]) + l * math.log(2 * math.pi)
    err = np.maximum(np.abs(d - o["d"]), np.abs(u - o["u"])) / scale
    jit = o["eps"] > 0
    assert np.max(err[~jit]) <= 1e-10, np.max(err[~jit])
    assert np.max(err[jit]) <= 1e-6, err[jit]
    assert abs(ll - o["loglik"]) <= 1e-8 * abs(o["loglik"]), (ll, o["loglik"])
    # an evaluation without failures resets the count and matches the mode-off result
    p = bvgen.make_plan("c1", n=400, bc=16, m=20, cfg=33)
    p = p.with_y(bvgen.normal(4402, p.n))
    a, b = BlockVecchia(p), BlockVecchia(p)
    b.set_jitter(True)
    assert a.loglik(theta) == b.loglik(theta) and b.jitter_events == 0
    bv.set_jitter(False)
    with pytest.raises(NotPositiveDefinite) as e:
        bv.loglik(theta)
    assert e.value.failed_position == 4


@pytest.mark.parametrize("shape", [dict(n=2000, bc=20, m=30, cfg=51), dict(n=6000, bc=150, m=60, cfg=52)])
def test_general_nu_pregeneration_is_bitwise_equal(shape, monkeypatch):
    """General ν on small plans: the all-SM pre-generation kernel + block kernel (KIND kPre)
    gives bitwise the ℓ, d_k, u_k of the in-kernel K_ν path (BV_NO_PREGEN=1): same
    function, same arguments, same order of the elimination."""
    theta = (1.1, 0.06, 0.83)
    p = bvgen.make_plan("c1", **shape)
    p = p.with_y(oracle.simulate_bv(p, theta, bvgen.normal(5101, p.n)))
    a = BlockVecchia(p)
    monkeypatch.setenv("BV_NO_PREGEN", "1")
    b = BlockVecchia(p)
    la, da, ua = a.loglik_terms(theta)
    lb, db, ub = b.loglik_terms(theta)
    assert a.launches_per_eval == b.launches_per_eval + 1
    assert la == lb and np.array_equal(da, db) and np.array_equal(ua, ub)
    o = oracle.bv_loglik(p, theta)
    assert abs(la - o["loglik"]) <= 1e-9 * abs(o["loglik"])


def test_jitter_mode_classic_vecchia_positions():
    """bc = n: a position whose point repeats its first neighbour fails in the warp kernel
    (bv_cv.cu, d_k = NaN marker) and is retried like any block (reading G15b)."""
    theta = (1.0, 0.078809, 1.5)
    n = 800
    p = bvgen.make_plan("c1", n=n, bc=n, m=25, cfg=38)
    pt = np.empty(n, dtype=np.int32)
    pt[p.block_id] = np.arange(n, dtype=np.int32)
    locs, y = p.locs.copy(), bvgen.normal(3803, n)
    for k in (300, 650):
        i = p.nbr_idx[p.nbr_ptr[k]]
        locs[pt[p.order[k]]] = locs[i]
        y[pt[p.order[k]]] = y[i] + 1e-6
    q = bvgen.Plan(locs, y, p.block_id, p.order, p.nbr_ptr, p.nbr_idx)
    o = oracle.bv_loglik_jitter(q, theta)
    assert o["events"] >= 2
    bv = BlockVecchia(q)
    with pytest.raises(NotPositiveDefinite) as e:
        bv.loglik(theta)
    assert e.value.failed_position == 300
    bv.set_jitter(True)
    ll, d, u = bv.loglik_terms(theta)
    assert bv.jitter_events == o["events"]
    scale = np.abs(o["u"]) + np.abs(o["d"]) + math.log(2 * math.pi)
    err = np.maximum(np.abs(d - o["d"]), np.abs(u - o["u"])) / scale
    jit = o["eps"] > 0
    assert np.max(err[~jit]) <= 1e-10 and np.max(err[jit]) <= 1e-6
    assert abs(ll - o["loglik"]) <= 1e-8 * abs(o["loglik"])
