"""Block-Vecchia prediction (Alg. 2; §2.3) — §8f row 1.

CPU (-m "not gpu"): the oracle's Alg. 2 pinned against what the mathematics fixes —
  * one prediction block conditioned on ALL training points = the exact GP conditional
    μ = Σ*y Σyy⁻¹ y, Σ = Σ** − Σ*y Σyy⁻¹ Σy* (the §2.3 formulas), computed here
    by LU solves (numpy), not Cholesky;
  * interpolation: a new location equal to a conditioning training location gets μ = y_i, var = 0;
  * far from every neighbour (r/β > 700): μ = 0 and Σ_B* = Σlk exactly; m = 0 likewise;
  * Σ_B* symmetric positive semi-definite, its diagonal = var.
GPU (-m gpu): bv_predict (one CTA per prediction block, Schur complement of the joint matrix
after eliminating the m neighbour columns) vs the oracle element by element.
"""
import numpy as np
import pytest

import bvgen
import oracle

THETAS = [(1.0, 0.1, 0.5), (1.3, 0.08, 1.5), (0.9, 0.12, 2.5), (1.1, 0.07, 1.2)]


def train_set(n=150, d=2, seed=71, theta=(1.0, 0.1, 1.5)):
    locs = bvgen.uniform(seed, n * d).reshape(n, d)
    y = oracle.simulate_exact(locs, theta, bvgen.normal(seed + 1, n))
    return locs, y


def cov_matrix(A, B, theta):
    return np.array([[oracle.matern(float(np.sqrt(np.sum((a - b) ** 2))), theta) for b in B] for a in A])


@pytest.mark.parametrize("theta", THETAS)
def test_oracle_predict_full_conditioning_is_exact(theta):
    locs, y = train_set(theta=theta)
    n = locs.shape[0]
    new = bvgen.uniform(79, 12 * 2).reshape(12, 2)
    ptr = np.array([0, n], dtype=np.int64)
    idx = np.arange(n, dtype=np.int32)[::-1].copy()  # any order of the conditioning set
    o = oracle.bv_predict(locs, y, theta, new, np.zeros(12, dtype=np.int32), ptr, idx, want_cov=True)
    Syy = cov_matrix(locs, locs, theta)
    Sxy = cov_matrix(new, locs, theta)
    Sxx = cov_matrix(new, new, theta)
    mu = Sxy @ np.linalg.solve(Syy, y)
    S = Sxx - Sxy @ np.linalg.solve(Syy, Sxy.T)
    scale = np.sqrt(theta[0]) + np.max(np.abs(mu))
    assert np.max(np.abs(o["mean"] - mu)) <= 1e-8 * scale
    assert np.max(np.abs(o["cov"].reshape(12, 12) - S)) <= 1e-8 * theta[0]
    np.testing.assert_array_equal(o["var"], np.diag(o["cov"].reshape(12, 12)))


def test_oracle_predict_interpolates_training_points():
    theta = (1.0, 0.1, 1.5)
    locs, y = train_set(theta=theta)
    pick = [3, 40, 77]
    new = locs[pick].copy()
    ptr = np.array([0, 20, 40, 60], dtype=np.int64)
    idx = []
    for b, i in enumerate(pick):  # the picked point plus 19 others
        others = [j for j in range(150) if j != i][b * 19:(b + 1) * 19]
        idx += [i] + others
    o = oracle.bv_predict(locs, y, theta, new, np.arange(3, dtype=np.int32), ptr, np.array(idx, dtype=np.int32))
    assert np.max(np.abs(o["mean"] - y[pick])) <= 1e-10 * np.max(np.abs(y))
    assert np.max(np.abs(o["var"])) <= 1e-10 * theta[0]


def test_oracle_predict_far_field_and_no_neighbours():
    theta = (1.7, 0.001, 0.5)
    locs, y = train_set(theta=(1.0, 0.1, 0.5))
    new = np.array([[5.0, 5.0], [5.0001, 5.0], [9.0, 1.0]])  # r/β > 4000 from every training point
    bid = np.array([0, 0, 1], dtype=np.int32)
    ptr = np.array([0, 10, 10], dtype=np.int64)  # block 1: m = 0
    o = oracle.bv_predict(locs, y, theta, new, bid, ptr, np.arange(10, dtype=np.int32), want_cov=True)
    assert np.all(o["mean"] == 0.0)
    lk = cov_matrix(new[:2], new[:2], theta)
    np.testing.assert_array_equal(o["cov"][:4].reshape(2, 2), lk)
    assert o["cov"][4] == theta[0] and np.all(o["var"] == theta[0])


def test_oracle_predict_cov_symmetric_psd():
    theta = (1.0, 0.06, 1.5)
    locs, y = train_set(n=400, theta=theta)
    pp = bvgen.make_pred_plan(locs, bvgen.uniform(83, 60 * 2).reshape(60, 2), 6, 25)
    o = oracle.bv_predict(locs, y, theta, pp.locs_new, pp.block_id, pp.nbr_ptr, pp.nbr_idx, want_cov=True)
    off = 0
    for b in range(6):
        mem = np.nonzero(pp.block_id == b)[0]
        lb = len(mem)
        S = o["cov"][off:off + lb * lb].reshape(lb, lb)
        off += lb * lb
        assert np.max(np.abs(S - S.T)) <= 1e-15
        assert np.min(np.linalg.eigvalsh(S)) >= -1e-12
        np.testing.assert_array_equal(np.diag(S), o["var"][mem])
        assert np.all(o["var"][mem] <= theta[0])  # conditioning never increases variance


def test_pred_plan_nn_matches_bruteforce():
    locs, _ = train_set(n=300)
    new = bvgen.uniform(91, 40 * 2).reshape(40, 2)
    pp = bvgen.make_pred_plan(locs, new, 5, 17)
    for b in range(5):
        c = new[pp.block_id == b].mean(axis=0)
        d2 = (locs[:, 0] - c[0]) ** 2 + (locs[:, 1] - c[1]) ** 2
        want = np.lexsort((np.arange(300), d2))[:17]
        np.testing.assert_array_equal(pp.nbr_idx[pp.nbr_ptr[b]:pp.nbr_ptr[b + 1]], want)


# ------------------------------------------------------------------------------------ GPU
def gpu_case(name, theta, n_new, bc_new, m, cfg):
    p = bvgen.make_plan(name, cfg=cfg)
    p = p.with_y(oracle.simulate_bv(p, theta, bvgen.normal(100 * cfg + 2, p.n)))
    new = bvgen.uniform(100 * cfg + 7, n_new * p.d).reshape(n_new, p.d)
    if p.d == 3:
        new[:, 2] = np.floor(new[:, 2] * 17.0) / 16.0
    return p, bvgen.make_pred_plan(p.locs, new, bc_new, m)


@pytest.mark.gpu
@pytest.mark.parametrize("name,theta,n_new,bc_new,m", [
    ("c1", (1.0, 0.078809, 0.5), 500, 50, 30),
    ("c1", (1.0, 0.078809, 1.5), 500, 20, 120),
    ("c2", (1.0, 0.052537, 1.5), 2000, 200, 60),
    ("c2", (0.9, 0.06, 1.31), 1000, 100, 60),
    ("c1", (1.0, 0.078809, 1.5), 300, 30, 31),  # odd m: the kernel's single-column tail step
    ("c1", (1.0, 0.078809, 2.5), 200, 20, 1),
])
def test_predict_gpu_parity(name, theta, n_new, bc_new, m):
    from paper_2410_04477_b200 import BlockVecchia
    p, pp = gpu_case(name, theta, n_new, bc_new, m, {"c1": 1, "c2": 2}[name])
    bv = BlockVecchia(p)
    mean, var, cov = bv.predict(theta, pp, want_cov=True)
    bv.close()
    o = oracle.bv_predict(p.locs, p.y, theta, pp.locs_new, pp.block_id, pp.nbr_ptr, pp.nbr_idx, want_cov=True)
    em = np.max(np.abs(mean - o["mean"])) / (np.sqrt(theta[0]) + np.max(np.abs(o["mean"])))
    ev = np.max(np.abs(var - o["var"])) / theta[0]
    ec = np.max(np.abs(cov - o["cov"])) / theta[0]
    print(name, theta, "mean", em, "var", ev, "cov", ec)
    assert em <= 1e-9 and ev <= 1e-9 and ec <= 1e-9


@pytest.mark.gpu
def test_predict_gpu_rejects_bad_plans():
    from paper_2410_04477_b200 import BlockVecchia, BVError
    p, pp = gpu_case("c1", (1.0, 0.078809, 0.5), 100, 10, 30, 1)
    bv = BlockVecchia(p)
    bad = bvgen.PredPlan(pp.locs_new, pp.block_id, pp.nbr_ptr, pp.nbr_idx.copy())
    bad.nbr_idx[0] = p.n  # out of range
    with pytest.raises(BVError):
        bv.predict((1.0, 0.078809, 0.5), bad)
    big = bvgen.make_pred_plan(p.locs, pp.locs_new, 1, 200)  # m + l = 300 > 235
    with pytest.raises(BVError):
        bv.predict((1.0, 0.078809, 0.5), big)
    # the handle's duplicate-neighbour table persists across calls: repeated predictions agree
    # bitwise, and a duplicate is still caught after successful calls
    m1, v1 = bv.predict((1.0, 0.078809, 0.5), pp)
    assert bv.last_kernel_ms() > 0.0
    m2, v2 = bv.predict((1.0, 0.078809, 0.5), pp)
    assert np.array_equal(m1, m2) and np.array_equal(v1, v2)
    dup = bvgen.PredPlan(pp.locs_new, pp.block_id, pp.nbr_ptr, pp.nbr_idx.copy())
    dup.nbr_idx[1] = dup.nbr_idx[0]
    with pytest.raises(BVError):
        bv.predict((1.0, 0.078809, 0.5), dup)
    bv.close()
