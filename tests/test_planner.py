"""Input-generator tests (-m "not gpu"): RNG, locations, K-means, block-NN.

The planner (bvgen/planner.cpp) is pinned bit-exact against the oracle's
O(n²) brute force and the brute-force Lloyd assignment.
"""
import numpy as np
import pytest

import bvgen
import oracle


def test_rng_is_deterministic_and_uniform():
    a = bvgen.uniform(5, 10000)
    assert np.array_equal(a, bvgen.uniform(5, 10000))
    assert a.min() >= 0 and a.max() < 1 and abs(a.mean() - 0.5) < 0.01
    assert np.array_equal(bvgen.uniform(5, 10, offset=100), bvgen.uniform(5, 110)[100:])
    z = bvgen.normal(6, 200000)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01


def test_permutation_is_bijection():
    for n in (1, 2, 17, 1000):
        p = bvgen.permutation(3, n)
        assert np.array_equal(np.sort(p), np.arange(n))


def test_c4_locations_have_17_levels():
    """c4: z = k/16, k ∈ {0..16} (reading G16)."""
    L = bvgen.locations(4, 20000, 3)
    assert np.array_equal(np.unique(L[:, 2]), np.arange(17) / 16.0)


@pytest.mark.parametrize("n,bc,m,d", [(300, 30, 10, 2), (500, 40, 25, 2), (400, 20, 60, 3), (200, 200, 5, 2),
                                      (120, 3, 100, 2)])
def test_block_nn_equals_bruteforce(n, bc, m, d):
    """Alg. 1 l.7-9: grid ring search == O(n²) brute force, bit-exact."""
    p = bvgen.make_plan("c4" if d == 3 else "c1", n=n, bc=bc, m=m, d=d, cfg=9)
    ptr, idx = oracle.block_nn_bruteforce(p.locs, p.block_id, p.order, m)
    assert np.array_equal(ptr, p.nbr_ptr)
    assert np.array_equal(idx, p.nbr_idx)


def test_block_nn_ties_on_lattice():
    """Exact ties (lattice points, layered z) are broken by global id."""
    g = np.stack(np.meshgrid(np.arange(12) / 11.0, np.arange(12) / 11.0, indexing="ij"), -1).reshape(-1, 2)
    block_id = (np.arange(144) % 16).astype(np.int32)
    order = bvgen.permutation(77, 16)
    ptr, idx = bvgen.block_nn(g, block_id, order, 13)
    bptr, bidx = oracle.block_nn_bruteforce(g, block_id, order, 13)
    assert np.array_equal(ptr, bptr) and np.array_equal(idx, bidx)


def test_neighbours_are_earlier_and_unique():
    p = bvgen.make_plan("c1", n=2000, bc=50, m=40, cfg=10)
    pos = np.empty(p.bc, dtype=np.int64)
    pos[p.order] = np.arange(p.bc)
    l, mk = p.block_sizes()
    before = np.concatenate([[0], np.cumsum(l)])[:-1]
    assert np.array_equal(mk, np.minimum(40, before))
    for k in range(p.bc):
        s = p.nbr_idx[p.nbr_ptr[k]:p.nbr_ptr[k + 1]]
        assert len(np.unique(s)) == len(s)
        assert np.all(pos[p.block_id[s]] < k)


def test_kmeans_assignment_equals_bruteforce():
    """One Lloyd step from the seeded init == brute-force nearest centroid (ties → lower id)."""
    for d, n, k in ((2, 3000, 60), (3, 3000, 50)):
        locs = bvgen.locations(4 if d == 3 else 1, n, d)
        init = bvgen.sample_without_replacement(31, n, k)
        assign, _, _ = bvgen.kmeans(locs, k, 31, max_iter=1)
        ref = oracle.kmeans_assign_bruteforce(locs, locs[init])
        assert np.array_equal(assign, ref)


def test_kmeans_partition_valid():
    """disjoint cover, no empty block."""
    locs = bvgen.locations(1, 5000, 2)
    assign, cent, it = bvgen.kmeans(locs, 100, 3, max_iter=100)
    cnt = np.bincount(assign, minlength=100)
    assert cnt.min() >= 1 and cnt.sum() == 5000
    for c in (0, 17, 99):
        assert np.allclose(cent[c], locs[assign == c].mean(0))


def test_kmeans_objective_nonincreasing():
    locs = bvgen.locations(1, 4000, 2)
    obj = []
    for it in (1, 2, 4, 8, 16):
        a, c, _ = bvgen.kmeans(locs, 80, 5, max_iter=it)
        obj.append(np.sum((locs - c[a]) ** 2))
    assert all(x >= y - 1e-12 for x, y in zip(obj, obj[1:])), obj
