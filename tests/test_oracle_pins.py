"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the passage it pins.  None of them re-types the oracle's own
formula: they use printed constants, reductions to other definitions
(Eq. 1 exact likelihood, classic Vecchia), invariances, metamorphic identities
and an independent formulation (joint-Cholesky simulation).
"""
import math
import os

import mpmath
import numpy as np
import pytest

import bvgen
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append([float(x) for x in line.split()])
    return rows


def small_plan(n=200, bc=10, m=12, d=2, cfg=7, theta=None, sim=True):
    p = bvgen.make_plan("c1", n=n, bc=bc, m=m, d=d, cfg=cfg)
    if sim and theta is not None:
        eps = bvgen.normal(100 * cfg + 2, n)
        p = p.with_y(oracle.simulate_bv(p, theta, eps))
    return p


THETAS = [(1.0, 0.1, 0.5), (2.0, 0.2, 1.5), (1.3, 0.15, 2.5), (0.7, 0.12, 0.83)]


# ------------------------------------------------------------------ constants
def test_ln_2pi_is_correctly_rounded():
    """Reading G23: ln 2π = 0x3FFD67F1C864BEB5 (mpmath at 50 digits)."""
    mpmath.mp.dps = 50
    assert oracle.ln_2pi() == float(mpmath.log(2 * mpmath.pi))


# ------------------------------------------------------------------ Matérn
def test_matern_closed_forms_at_x1():
    """Eq. (7) at x=1 vs SPEC.md:130-132 printed values (3rd corrected), golden file."""
    beta = 0.0731
    for nu, val, tol in _golden("matern_x1.txt"):
        got = oracle.matern([beta], (1.0, beta, nu))[0]
        assert abs(got - val) <= tol * val, (nu, got, val)


def test_matern_zero_distance_is_sigma2():
    """C(0) = σ² (continuous limit of Eq. 7)."""
    for nu in (0.5, 1.5, 2.5, 0.83, 3.7):
        assert oracle.matern([0.0], (2.5, 0.1, nu))[0] == 2.5


@pytest.mark.parametrize("nu", [0.5, 1.5, 2.5])
def test_matern_general_path_reduces_to_closed_forms(nu):
    """The general K_ν path of Eq. (7) equals the elementary forms at half-integer ν (≤1e-13)."""
    beta = 0.05
    x = np.geomspace(1e-6, 40, 300)
    r = x * beta
    closed = oracle.matern(r, (1.0, beta, nu), mode=0)
    general = oracle.matern(r, (1.0, beta, nu), mode=1)
    rel = np.abs(general - closed) / np.abs(closed)
    assert rel.max() <= 1e-13, rel.max()


def test_matern_general_nu_vs_mpmath():
    """General ν: Eq. (7) against mpmath's besselk/gamma at 40 digits."""
    mpmath.mp.dps = 40
    rng = np.random.default_rng(5)
    for _ in range(60):
        nu = float(rng.uniform(0.2, 4.0))
        x = float(np.exp(rng.uniform(np.log(1e-4), np.log(40.0))))
        beta = 0.07
        ref = 2 ** (1 - mpmath.mpf(nu)) / mpmath.gamma(nu) * mpmath.mpf(x) ** nu * mpmath.besselk(nu, x)
        got = oracle.matern([x * beta], (1.0, beta, nu), mode=1)[0]
        # x*beta/beta may differ from x by an ulp; compare at the oracle's own x
        xo = (x * beta) / beta
        ref = 2 ** (1 - mpmath.mpf(nu)) / mpmath.gamma(nu) * mpmath.mpf(xo) ** nu * mpmath.besselk(nu, xo)
        assert abs(got - float(ref)) <= 1e-13 * abs(float(ref)), (nu, x, got, float(ref))


def test_table1_effective_range_convention():
    """Table 1 β values all give C(range)/σ² = 0.02222 ± 1e-5 under x = r/β (G2, G3)."""
    for nu, rng_, beta in _golden("table1_beta.txt"):
        c = oracle.matern([rng_], (1.0, beta, nu))[0]
        assert abs(c - 0.022222) <= 1e-5, (nu, rng_, beta, c)


def test_matern_monotone_and_bounded():
    """0 < C(r) ≤ σ², non-increasing in r."""
    r = np.linspace(0, 1.5, 400)
    for th in THETAS:
        c = oracle.matern(r, th)
        assert np.all(np.diff(c) <= 0) and c[0] == th[0] and np.all(c >= 0)


# ------------------------------------------------------------------ dense primitives
def test_cholesky_hand_example():
    """[[4,2],[2,3]] → [[2,0],[1,√2]]."""
    L = oracle.potrf(np.array([[4.0, 2.0], [2.0, 3.0]]))
    assert np.allclose(L, [[2, 0], [1, math.sqrt(2)]], rtol=0, atol=1e-15)


def test_cholesky_and_trsv_residuals():
    """‖LLᵀ−A‖ and ‖Lx−b‖ small on random SPD matrices."""
    rng = np.random.default_rng(1)
    for n in (1, 5, 17, 64):
        G = rng.standard_normal((n, n))
        A = G @ G.T + n * np.eye(n)
        L = oracle.potrf(A)
        assert np.allclose(np.triu(L, 1), 0)
        assert np.linalg.norm(L @ L.T - A) <= 1e-13 * np.linalg.norm(A)
        b = rng.standard_normal(n)
        x = oracle.trsv(L, b)
        assert np.abs(L @ x - b).max() <= 1e-12 * np.abs(b).max()


def test_cholesky_rejects_non_pd():
    with pytest.raises(oracle.OracleError):
        oracle.potrf(np.array([[1.0, 1.0], [1.0, 1.0]]))


# ------------------------------------------------------------------ likelihood reductions
@pytest.mark.parametrize("theta", THETAS)
def test_single_block_equals_exact_likelihood(theta):
    """bc = 1: Eq. (4) collapses to Eq. (1)."""
    p = small_plan(n=80, bc=1, m=10, theta=None, sim=False)
    p = p.with_y(oracle.simulate_exact(p.locs, theta, bvgen.normal(11, p.n)))
    bv = oracle.bv_loglik(p, theta)["loglik"]
    ex = oracle.exact_loglik(p.locs, p.y, theta)
    assert abs(bv - ex) <= 1e-10 * abs(ex), (bv, ex)


def _full_conditioning(p):
    """Neighbour sets = every point of every earlier block (ascending id)."""
    pos = np.empty(p.bc, dtype=np.int64)
    pos[p.order] = np.arange(p.bc)
    ppos = pos[p.block_id]
    ptr = [0]
    idx = []
    for k in range(p.bc):
        earlier = np.where(ppos < k)[0]
        idx.extend(earlier.tolist())
        ptr.append(len(idx))
    return bvgen.Plan(p.locs, p.y, p.block_id, p.order, np.array(ptr, dtype=np.int64),
                      np.array(idx, dtype=np.int32))


@pytest.mark.parametrize("theta", THETAS)
def test_full_conditioning_equals_exact_likelihood(theta):
    """m_i = all earlier points: Eqs. (2)-(3) chain rule is exact."""
    p = small_plan(n=90, bc=7, m=5, sim=False)
    p = _full_conditioning(p).with_y(oracle.simulate_exact(p.locs, theta, bvgen.normal(12, p.n)))
    bv = oracle.bv_loglik(p, theta)["loglik"]
    ex = oracle.exact_loglik(p.locs, p.y, theta, long_double=True)
    assert abs(bv - ex) <= 1e-9 * abs(ex) + 1e-10, (bv, ex)


def test_full_conditioning_permutation_invariance():
    """Eq. (3): any permutation ζ gives the same joint density."""
    theta = (1.0, 0.1, 1.5)
    p = small_plan(n=90, bc=9, m=5, sim=False)
    p = p.with_y(oracle.simulate_exact(p.locs, theta, bvgen.normal(13, p.n)))
    vals = []
    for s in range(4):
        q = bvgen.Plan(p.locs, p.y, p.block_id, bvgen.permutation(900 + s, p.bc), p.nbr_ptr, p.nbr_idx)
        vals.append(oracle.bv_loglik(_full_conditioning(q), theta)["loglik"])
    assert max(vals) - min(vals) <= 1e-10 * abs(vals[0]), vals


@pytest.mark.parametrize("theta", THETAS)
def test_block_size_one_equals_classic_vecchia(theta):
    """bc = n: block Vecchia is classic Vecchia, solved independently by GEPP."""
    n = 150
    p = small_plan(n=n, bc=n, m=8, sim=False)
    p = p.with_y(oracle.simulate_exact(p.locs, theta, bvgen.normal(14, n)))
    bv = oracle.bv_loglik(p, theta)["loglik"]
    # classic Vecchia over points in ζ order: singleton block order[k] holds exactly one point
    pt = np.empty(n, dtype=np.int32)
    pt[p.block_id] = np.arange(n, dtype=np.int32)
    point_order = pt[p.order]
    cv = oracle.classic_vecchia(p.locs, p.y, point_order, p.nbr_ptr, p.nbr_idx, theta)
    assert abs(bv - cv) <= 1e-10 * abs(cv), (bv, cv)


def test_kl_nonnegative_and_nonincreasing_in_m():
    """Eq. (6): KL = ℓ0(θ;0) − ℓa(θ;0) ≥ 0, shrinking for nested neighbour sets."""
    theta = (1.0, 0.1, 1.5)
    base = small_plan(n=200, bc=20, m=40, sim=False, cfg=8)
    ex0 = oracle.exact_loglik(base.locs, np.zeros(base.n), theta)
    kls = []
    for m in (2, 5, 10, 20, 40):
        ptr = [0]
        idx = []
        for k in range(base.bc):
            s = base.nbr_idx[base.nbr_ptr[k]:base.nbr_ptr[k + 1]][:m]  # nested: first m keys
            idx.extend(s.tolist())
            ptr.append(len(idx))
        q = bvgen.Plan(base.locs, np.zeros(base.n), base.block_id, base.order, np.array(ptr, dtype=np.int64),
                       np.array(idx, dtype=np.int32))
        kls.append(ex0 - oracle.bv_loglik(q, theta)["loglik"])
    assert all(k >= -1e-10 for k in kls), kls
    assert all(a >= b - 1e-10 for a, b in zip(kls, kls[1:])), kls


# ------------------------------------------------------------------ metamorphic
def test_sigma2_scaling_is_exact():
    """Eq. (7) homogeneity: σ²→4σ² gives u/4 bitwise and d + 2 l ln 2."""
    theta = (1.0, 0.06, 1.5)
    p = small_plan(n=300, bc=15, m=20, theta=theta)
    a = oracle.bv_loglik(p, theta)
    b = oracle.bv_loglik(p, (4.0, 0.06, 1.5))
    l, _ = p.block_sizes()
    assert np.array_equal(b["u"], a["u"] / 4)
    shift = b["d"] - a["d"] - 2 * l * math.log(2.0)
    assert np.all(np.abs(shift) <= 1e-13 * (np.abs(a["d"]) + l))


def test_length_scaling_is_exact():
    """Isotropy in r/β: (coords, β) × 2^k leaves (u, d) bitwise unchanged."""
    theta = (1.0, 0.06, 2.5)
    p = small_plan(n=300, bc=15, m=20, theta=theta)
    a = oracle.bv_loglik(p, theta)
    for k in (3, -5):
        q = bvgen.Plan(p.locs * 2.0 ** k, p.y, p.block_id, p.order, p.nbr_ptr, p.nbr_idx)
        b = oracle.bv_loglik(q, (1.0, 0.06 * 2.0 ** k, 2.5))
        assert np.array_equal(a["u"], b["u"]) and np.array_equal(a["d"], b["d"])


# ------------------------------------------------------------------ generating model
def test_generating_model_pin():
    """y simulated block-sequentially (joint-Cholesky formulation) ⇒ v_i = ε_i, so u_i = ‖ε_i‖² and Σu ~ χ²_n."""
    theta = (1.0, 0.078809, 0.5)
    p = bvgen.make_plan("c1")
    eps = bvgen.normal(102, p.n)
    p = p.with_y(oracle.simulate_bv(p, theta, eps))
    r = oracle.bv_loglik(p, theta)
    e2 = np.array([np.sum(eps[np.where(p.block_id == b)[0]] ** 2) for b in p.order])
    assert np.max(np.abs(r["u"] - e2) / e2) <= 1e-12
    n = p.n
    assert abs(r["u"].sum() - n) <= 5 * math.sqrt(2 * n)


def test_long_double_agrees_at_c1():
    """FP64 Alg. 1 vs the 80-bit instance at c1: well-conditioned (κ ≲ 2e3), so ≤ 1e-12."""
    theta = (1.0, 0.078809, 0.5)
    p = bvgen.make_plan("c1")
    p = p.with_y(oracle.simulate_bv(p, theta, bvgen.normal(102, p.n)))
    a = oracle.bv_loglik(p, theta)
    b = oracle.bv_loglik(p, theta, long_double=True)
    assert abs(a["loglik"] - b["loglik"]) <= 1e-12 * abs(b["loglik"])
    s = np.abs(b["u"]) + np.abs(b["d"]) + p.block_sizes()[0] * oracle.ln_2pi()
    assert np.max(np.abs(a["t"] - b["t"]) / s) <= 1e-13


def test_thread_count_determinism():
    """SPEC.md:316 / acceptance 9: bitwise identical across thread counts."""
    theta = (1.0, 0.05, 1.5)
    p = small_plan(n=2000, bc=40, m=30, theta=theta)
    a = oracle.bv_loglik(p, theta, nthreads=1)
    b = oracle.bv_loglik(p, theta, nthreads=5)
    assert a["loglik"] == b["loglik"] and np.array_equal(a["t"], b["t"])


def test_position_range_partial_sums_compose():
    """Σ over [0,k) + Σ over [k,bc) = the full per-block vector (used for the multi-GPU split)."""
    theta = (1.0, 0.05, 1.5)
    p = small_plan(n=1000, bc=25, m=20, theta=theta)
    full = oracle.bv_loglik(p, theta)
    a = oracle.bv_loglik(p, theta, k_range=(0, 11))
    b = oracle.bv_loglik(p, theta, k_range=(11, 25))
    assert np.array_equal(np.concatenate([a["t"], b["t"]]), full["t"])


def test_duplicate_points_are_not_pd():
    """Reading G15: a repeated location makes Σ singular → NOT_PD naming the smallest failing position."""
    theta = (1.0, 0.1, 0.5)
    p = small_plan(n=200, bc=10, m=10, sim=False)
    locs = p.locs.copy()
    b = p.order[4]
    members = np.where(p.block_id == b)[0]
    locs[members[1]] = locs[members[0]]
    q = bvgen.Plan(locs, p.y, p.block_id, p.order, p.nbr_ptr, p.nbr_idx)
    with pytest.raises(oracle.OracleError) as e:
        oracle.bv_loglik(q, theta)
    assert e.value.status == 3 and 0 <= e.value.failed_position <= 4


def test_invalid_theta_rejected():
    p = small_plan(n=100, bc=5, m=5, sim=False)
    for th in [(0.0, 0.1, 0.5), (1.0, -0.1, 0.5), (1.0, 0.1, float("nan"))]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.bv_loglik(p, th)
        assert e.value.status == 2


def test_perturbed_replicas_measure_fp64_error_at_high_kappa():
    """Reading G22: ±1-ulp entry replicas spread by ≈ FP64's own error; well-conditioned
    blocks barely move (c1, κ ≲ 2e3), and the spread never exceeds the long-double gap by orders."""
    theta = (1.0, 0.078809, 0.5)
    p = bvgen.make_plan("c1")
    p = p.with_y(oracle.simulate_bv(p, theta, bvgen.normal(102, p.n)))
    ld = oracle.bv_loglik(p, theta, long_double=True)
    l, _ = p.block_sizes()
    s = np.abs(ld["u"]) + np.abs(ld["d"]) + l * oracle.ln_2pi()
    for seed in (1, 2, 3):
        r = oracle.bv_loglik(p, theta, perturb_seed=seed)
        assert np.max(np.abs(r["t"] - ld["t"]) / s) <= 1e-13
    a = oracle.bv_loglik(p, theta, perturb_seed=1)
    b = oracle.bv_loglik(p, theta, perturb_seed=1)
    assert np.array_equal(a["t"], b["t"])  # deterministic


# ------------------------------------------------------------------ optional jitter mode (reading G15b)
def _exp_cov(A, B, theta):
    """ν = 1/2 Matérn written out: σ² exp(−r/β) (Eq. (7) at ν = 1/2)."""
    r = np.sqrt(((A[:, None, :] - B[None, :, :]) ** 2).sum(-1))
    return theta[0] * np.exp(-r / theta[1])


def _gauss_logpdf(S, y):
    Lc = np.linalg.cholesky(S)
    z = np.linalg.solve(Lc, y)
    return -0.5 * (z @ z + 2.0 * np.log(np.diag(Lc)).sum() + len(y) * math.log(2 * math.pi))


def _dup_plan(pos=4, n=200, bc=10, m=10):
    p = small_plan(n=n, bc=bc, m=m, sim=False)
    locs = p.locs.copy()
    b = p.order[pos]
    members = np.where(p.block_id == b)[0]
    locs[members[1]] = locs[members[0]]
    y = bvgen.normal(77, p.n)
    y[members[1]] = y[members[0]] + 1e-6
    return bvgen.Plan(locs, y, p.block_id, p.order, p.nbr_ptr, p.nbr_idx)


def test_jitter_single_block_equals_exact_likelihood_with_nugget():
    """bc = 1 with a repeated location: the jitter mode's first ε (1e-10)
    makes ℓ the exact Eq. (1) likelihood of Σθ + 1e-10·σ²·I (numpy dense Cholesky)."""
    theta = (1.3, 0.1, 0.5)
    p = small_plan(n=60, bc=1, m=5, sim=False)
    locs = p.locs.copy()
    locs[7] = locs[3]
    y = bvgen.normal(5, p.n)
    y[7] = y[3] + 1e-5
    q = bvgen.Plan(locs, y, p.block_id, p.order, p.nbr_ptr, p.nbr_idx)
    with pytest.raises(oracle.OracleError):
        oracle.bv_loglik(q, theta)
    r = oracle.bv_loglik_jitter(q, theta)
    S = _exp_cov(locs, locs, theta) + 1e-10 * theta[0] * np.eye(p.n)
    ex = _gauss_logpdf(S, y)
    assert r["events"] == 1 and r["eps"][0] == 1e-10
    assert abs(r["loglik"] - ex) <= 1e-7 * abs(ex), (r["loglik"], ex)


def test_jitter_blocks_equal_jittered_conditional_density():
    """Multi-block plan, one repeated location: every block that needed jitter has
    t_k = log p(y_NN, y_B) − log p(y_NN) under Σθ + ε·σ²·I (Eq. (4)'s conditional,
    PAPER.md:161, formed from two dense log-densities, not Alg. 1's steps); every
    other block is untouched (bitwise equal to Alg. 1 without jitter)."""
    theta = (1.0, 0.1, 0.5)
    q = _dup_plan()
    with pytest.raises(oracle.OracleError) as e:
        oracle.bv_loglik(q, theta)
    r = oracle.bv_loglik_jitter(q, theta)
    jit = np.nonzero(r["eps"])[0]
    assert r["events"] == len(jit) >= 1 and jit[0] == e.value.failed_position
    assert set(r["eps"][jit]) <= {1e-10, 1e-8, 1e-6}
    for k in range(q.bc):
        B = np.sort(np.where(q.block_id == q.order[k])[0])
        NN = q.nbr_idx[q.nbr_ptr[k]:q.nbr_ptr[k + 1]]
        if r["eps"][k] == 0:
            o = oracle.bv_loglik(q, theta, k_range=(k, k + 1))
            assert o["t"][0] == r["t"][k]
            continue
        J = np.concatenate([NN, B])
        SJ = _exp_cov(q.locs[J], q.locs[J], theta) + r["eps"][k] * theta[0] * np.eye(len(J))
        want = _gauss_logpdf(SJ, q.y[J])
        if len(NN):
            want -= _gauss_logpdf(SJ[:len(NN), :len(NN)], q.y[NN])
        assert abs(r["t"][k] - want) <= 1e-6 * (abs(want) + len(B)), (k, r["t"][k], want)
    assert abs(r["loglik"] - r["t"].sum()) <= 1e-9 * abs(r["loglik"])


def test_jitter_mode_is_identity_without_failures():
    """No failing block → the jitter mode returns Alg. 1's result bitwise, 0 events."""
    theta = THETAS[1]
    p = small_plan(n=300, bc=12, m=15, theta=theta)
    a = oracle.bv_loglik(p, theta)
    b = oracle.bv_loglik_jitter(p, theta)
    assert b["events"] == 0 and not b["eps"].any()
    assert a["loglik"] == b["loglik"] and np.array_equal(a["t"], b["t"])


def test_joint_formulation_diagnostic_agrees_in_long_double():
    """The diagnostic joint-Cholesky formulation (oracle.bv_loglik_joint, used only by
    tools/parity_diag.py) is exact arithmetic's same quantity: in 80-bit it equals Alg. 1 literal
    to rounding; in FP64 it differs by the formulation's own rounding."""
    theta = (1.0, 0.09, 1.5)
    p = bvgen.make_plan("c1", n=600, bc=12, m=24, cfg=41)
    p = p.with_y(oracle.simulate_bv(p, theta, bvgen.normal(4102, p.n)))
    a = oracle.bv_loglik(p, theta, long_double=True)
    b = oracle.bv_loglik_joint(p, theta, long_double=True)
    sc = np.abs(a["u"]) + np.abs(a["d"]) + 1.0
    assert np.max(np.abs(a["u"] - b["u"]) / sc) < 1e-13 and np.max(np.abs(a["d"] - b["d"]) / sc) < 1e-13
    assert abs(a["loglik"] - b["loglik"]) <= 1e-13 * abs(a["loglik"])


def test_simulate_exact_is_the_cholesky_draw():
    """or_simulate_exact draws y = L ε with L L ᵀ = Σ(θ): then yᵀΣ⁻¹y = ‖ε‖², so Eq. (1) at y plus
    ½‖ε‖² is the same number −½(log|Σ| + n log 2π) for every ε (pinned against exact_loglik, itself
    pinned by the Cholesky hand example and the bc = 1 reduction).  A wrong factor (transposed, not
    the Cholesky of Σ) breaks the identity."""
    theta = (1.3, 0.12, 1.5)
    locs = bvgen.locations(77, 300, 2)
    vals = []
    for seed in (1, 2, 3):
        eps = bvgen.normal(7700 + seed, 300)
        y = oracle.simulate_exact(locs, theta, eps)
        vals.append(oracle.exact_loglik(locs, y, theta) + 0.5 * float(eps @ eps))
    assert max(vals) - min(vals) <= 1e-9 * abs(vals[0]), vals
    # and y = 0·ε gives exactly that constant
    z = oracle.exact_loglik(locs, oracle.simulate_exact(locs, theta, np.zeros(300)), theta)
    assert abs(z - vals[0]) <= 1e-9 * abs(z)
