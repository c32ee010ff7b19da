"""GPU plan construction (bv_plan_kmeans / bv_plan_block_nn; Alg. 1 l.4-9, PAPER.md:586-591;
SURVEY §8f row 2): bit-identical to the CPU planner (bvgen/planner.cpp — an independent grid/heap
implementation, itself pinned against O(n²) brute force in tests/test_planner.py)."""
import time

import numpy as np
import pytest

import bvgen

pytestmark = pytest.mark.gpu


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
