"""GPU plan construction (bv_plan_kmeans / bv_plan_block_nn; Alg. 1 l.4-9, PAPER.md:586-591;
SURVEY §8f row 2): bit-identical to the oracle's O(n²) brute force (the selection exactly as
PAPER.md:104, :165, :589-591 define it, ties by (d², id)) on small inputs including lattice ties,
and to the CPU planner (bvgen/planner.cpp) at config sizes."""
import time

import numpy as np
import pytest

import bvgen
import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,bc,m,d", [(300, 30, 10, 2), (500, 40, 25, 2), (400, 20, 60, 3), (200, 200, 5, 2),
                                      (120, 3, 100, 2), (500, 25, 40, 3)])
def test_gpu_block_nn_equals_oracle_bruteforce(n, bc, m, d):
    """Alg. 1 l.7-9: the GPU's neighbour lists == the oracle's O(n²) brute force, bit-exact."""
    from paper_2410_04477_b200 import gpu_block_nn
    p = bvgen.make_plan("c4" if d == 3 else "c1", n=n, bc=bc, m=m, d=d, cfg=9)
    ptr, idx = gpu_block_nn(p.locs, p.block_id, p.order, m)
    bptr, bidx = oracle.block_nn_bruteforce(p.locs, p.block_id, p.order, m)
    np.testing.assert_array_equal(ptr, bptr)
    np.testing.assert_array_equal(idx, bidx)


def test_gpu_block_nn_lattice_ties():
    """Exact distance ties (a 12×12 lattice; a 3D lattice of 5 layers) are broken by global id
    exactly as the brute force does."""
    from paper_2410_04477_b200 import gpu_block_nn
    g2 = np.stack(np.meshgrid(np.arange(12) / 11.0, np.arange(12) / 11.0, indexing="ij"), -1).reshape(-1, 2)
    g3 = np.stack(np.meshgrid(np.arange(6) / 5.0, np.arange(6) / 5.0, np.arange(5) / 4.0, indexing="ij"),
                  -1).reshape(-1, 3)
    for g, nb, m in ((g2, 16, 13), (g3, 20, 30)):
        block_id = (np.arange(len(g)) % nb).astype(np.int32)
        order = bvgen.permutation(77, nb)
        ptr, idx = gpu_block_nn(g, block_id, order, m)
        bptr, bidx = oracle.block_nn_bruteforce(g, block_id, order, m)
        np.testing.assert_array_equal(ptr, bptr)
        np.testing.assert_array_equal(idx, bidx)


def test_gpu_kmeans_step_equals_oracle_assignment():
    """One Lloyd step on the GPU from the seeded init == the oracle's brute-force nearest centroid
    (ties → lower centroid id), incl. a lattice where many points are
    equidistant from two centroids."""
    from paper_2410_04477_b200 import gpu_kmeans
    for d, n, k in ((2, 3000, 60), (3, 3000, 50)):
        locs = bvgen.locations(4 if d == 3 else 1, n, d)
        init = bvgen.sample_without_replacement(31, n, k)
        assign, _, _ = gpu_kmeans(locs, k, init, max_iter=1)
        np.testing.assert_array_equal(assign, oracle.kmeans_assign_bruteforce(locs, locs[init]))
    g = np.stack(np.meshgrid(np.arange(16) / 15.0, np.arange(16) / 15.0, indexing="ij"), -1).reshape(-1, 2)
    init = (np.arange(0, 256, 17) % 256).astype(np.int32)  # lattice points as centroids: many exact ties
    assign, _, _ = gpu_kmeans(g, len(init), init, max_iter=1)
    np.testing.assert_array_equal(assign, oracle.kmeans_assign_bruteforce(g, g[init]))


@pytest.mark.parametrize("name,n,bc,m,d", [
    ("c1", 2000, 20, 30, 2),
    ("c2", 20000, 500, 60, 2),
    ("c4", 30000, 1500, 100, 3),   # 17 z-layers: many exact distance ties across layers
    ("c1", 500, 500, 10, 2),       # bc = n (classic Vecchia plans)
    ("c5", 50000, 2500, 200, 2),
])
def test_gpu_planner_bit_exact(name, n, bc, m, d):
    from paper_2410_04477_b200 import gpu_kmeans, gpu_block_nn
    cfg = bvgen.CONFIGS[name]["cfg"]
    locs = bvgen.locations(cfg, n, d)
    init = bvgen.sample_without_replacement(100 * cfg + 3, n, bc)
    iters = 100 if n <= 20000 else 20
    a_cpu, c_cpu, it_cpu = bvgen.kmeans(locs, bc, 100 * cfg + 3, iters)
    a_gpu, c_gpu, it_gpu = gpu_kmeans(locs, bc, init, iters)
    assert it_gpu == it_cpu
    np.testing.assert_array_equal(a_gpu, a_cpu)
    assert np.array_equal(c_gpu.view(np.uint64), c_cpu.view(np.uint64))  # bitwise
    order = bvgen.permutation(100 * cfg + 4, bc)
    p_cpu, i_cpu = bvgen.block_nn(locs, a_cpu, order, m)
    p_gpu, i_gpu = gpu_block_nn(locs, a_cpu, order, m)
    np.testing.assert_array_equal(p_gpu, p_cpu)
    np.testing.assert_array_equal(i_gpu, i_cpu)


def test_gpu_planner_full_c4_timed():
    """c4 at full size (n = 1M, 50k blocks, m = 100): identical NN lists, timings reported."""
    from paper_2410_04477_b200 import gpu_kmeans, gpu_block_nn
    c = bvgen.CONFIGS["c4"]
    locs = bvgen.locations(c["cfg"], c["n"], c["d"])
    init = bvgen.sample_without_replacement(100 * c["cfg"] + 3, c["n"], c["bc"])
    t = time.perf_counter()
    a_cpu, _, _ = bvgen.kmeans(locs, c["bc"], 100 * c["cfg"] + 3, 20)
    t_cpu_km = time.perf_counter() - t
    t = time.perf_counter()
    a_gpu, _, _ = gpu_kmeans(locs, c["bc"], init, 20)
    t_gpu_km = time.perf_counter() - t
    np.testing.assert_array_equal(a_gpu, a_cpu)
    order = bvgen.permutation(100 * c["cfg"] + 4, c["bc"])
    t = time.perf_counter()
    p_cpu, i_cpu = bvgen.block_nn(locs, a_cpu, order, c["m"])
    t_cpu_nn = time.perf_counter() - t
    t = time.perf_counter()
    p_gpu, i_gpu = gpu_block_nn(locs, a_cpu, order, c["m"])
    t_gpu_nn = time.perf_counter() - t
    np.testing.assert_array_equal(i_gpu, i_cpu)
    print(f"c4 planner: K-means CPU {t_cpu_km:.2f}s GPU {t_gpu_km:.2f}s; block-NN CPU {t_cpu_nn:.2f}s GPU {t_gpu_nn:.2f}s")


def test_gpu_planner_rejects_bad_input():
    from paper_2410_04477_b200 import gpu_block_nn, BVError
    locs = bvgen.locations(1, 100, 2)
    with pytest.raises(BVError):
        gpu_block_nn(locs, np.zeros(100, dtype=np.int32), np.array([0, 0], dtype=np.int32), 5)
    with pytest.raises(BVError):
        gpu_block_nn(locs, np.zeros(100, dtype=np.int32), np.array([0], dtype=np.int32), 300)
