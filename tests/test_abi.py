"""C-ABI tests that run without a GPU (-m "not gpu").

* libbv.so loads and exports every function include/bv.h declares;
* bv_setup's validation rejects bad plans (it runs before any CUDA call);
* the host-side twins: cost-balanced partition and the exact fixed-point
  encoding of block terms.
"""
import math
import os
import re
from fractions import Fraction

import numpy as np
import pytest

import bvgen
import paper_2410_04477_b200 as bvl
from paper_2410_04477_b200 import build as bvbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    bvbuild.build()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "bv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bv_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(bvl.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = bvl.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    assert b"sm_100a" in L.bv_version()


def test_built_for_sm100a():
    out = os.popen(f"cuobjdump --list-elf {bvl.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def _plan(n=300, bc=12, m=10):
    return bvgen.make_plan("c1", n=n, bc=bc, m=m, cfg=21)


def _setup_status(plan):
    try:
        bvl.BlockVecchia(plan)
    except bvl.BVError as e:
        return e.status, str(e)
    return 0, ""


@pytest.mark.parametrize("mutate,needle", [
    (lambda p: setattr(p, "order", np.zeros_like(p.order)), "permutation"),
    (lambda p: p.block_id.__setitem__(3, p.bc), "out of range"),
    (lambda p: p.locs.__setitem__((5, 0), np.nan), "not finite"),
    (lambda p: p.y.__setitem__(7, np.inf), "not finite"),
])
def test_setup_rejects_invalid_plans(mutate, needle):
    p = _plan()
    p.locs = p.locs.copy()
    p.y = p.y.copy()
    p.block_id = p.block_id.copy()
    mutate(p)
    st, msg = _setup_status(p)
    assert st == bvl.BV_EINVAL and needle in msg, msg


def test_setup_rejects_later_block_neighbour():
    p = _plan()
    idx = p.nbr_idx.copy()
    k = 5
    later_block = p.order[k]  # a point of the block itself is not "earlier"
    idx[p.nbr_ptr[k]] = int(np.where(p.block_id == later_block)[0][0])
    p.nbr_idx = idx
    st, msg = _setup_status(p)
    assert st == bvl.BV_EINVAL and "earlier" in msg, msg


def test_setup_rejects_duplicate_neighbour():
    p = _plan()
    idx = p.nbr_idx.copy()
    k = 6
    idx[p.nbr_ptr[k] + 1] = idx[p.nbr_ptr[k]]
    p.nbr_idx = idx
    st, msg = _setup_status(p)
    assert st == bvl.BV_EINVAL and "duplicate" in msg, msg


def test_setup_rejects_empty_block():
    p = _plan()
    bid = p.block_id.copy()
    bid[bid == p.order[3]] = p.order[2]
    p.block_id = bid
    st, msg = _setup_status(p)
    assert st == bvl.BV_EINVAL and "empty" in msg, msg


# ---------------------------------------------------------------- partition twin
def partition_twin(l, m, world):
    """Python restatement of bv_partition (include/bv.h): same double arithmetic, same order."""
    bc = len(l)
    prefix = [0.0]
    for k in range(bc):
        N = float(l[k]) + float(m[k])
        cost = N * N * N / 3.0 + 40.0 * (N * (N + 1.0) / 2.0)
        prefix.append(prefix[-1] + cost)
    total = prefix[-1]
    cuts = [0]
    k = 0
    for g in range(1, world):
        target = float(g) * total / float(world)
        while k < bc and prefix[k] < target:
            k += 1
        cuts.append(k)
    cuts.append(bc)
    return np.array(cuts, dtype=np.int32)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_partition_matches_twin_and_balances(world):
    p = bvgen.make_plan("c1", n=20000, bc=500, m=60, cfg=2)
    l, m = p.block_sizes()
    cuts = bvl.partition(l, m, world)
    assert np.array_equal(cuts, partition_twin(l, m, world))
    assert cuts[0] == 0 and cuts[-1] == p.bc and np.all(np.diff(cuts) >= 0)
    N = (l + m).astype(float)
    cost = N ** 3 / 3 + 40 * N * (N + 1) / 2
    shares = [cost[cuts[g]:cuts[g + 1]].sum() for g in range(world)]
    assert max(shares) <= cost.sum() / world + cost.max() + 1e-6


def test_partition_more_ranks_than_blocks():
    cuts = bvl.partition([3, 4], [0, 2], 5)
    assert cuts[0] == 0 and cuts[-1] == 2 and np.all(np.diff(cuts) >= 0)


# ---------------------------------------------------------------- fixed point
def _exact(t):
    """round(t·2⁶⁴) as a Python int (round half to even), via Fraction."""
    f = Fraction(t) * (1 << 64)
    return round(f)


def _chunks_to_int(c):
    v = sum(int(x) << (32 * i) for i, x in enumerate(c))
    return v - (1 << 192) if v >> 191 else v


@pytest.mark.parametrize("t", [0.0, -0.0, 1.0, -1.0, 0.5, -1234.5678, 1e-25, -3e-20, 2.0 ** -65, 2.0 ** -66 * 3,
                               7.9e28, -7.9e28, math.pi * 1e6, 5e-324])
def test_fixed_encode_is_round_t_times_2_64(t):
    c = bvl.fixed_encode(t)
    assert _chunks_to_int(c) == _exact(t)


def test_fixed_encode_rejects_out_of_range():
    for t in (2.0 ** 96, -(2.0 ** 97), float("inf"), float("nan")):
        with pytest.raises(bvl.BVError):
            bvl.fixed_encode(t)


def test_fixed_sum_is_order_independent_and_exact():
    rng = np.random.default_rng(3)
    t = -0.5 * (rng.gamma(20, 1, 5000) + rng.normal(-30, 20, 5000) + 20 * 1.8378770664093456)
    chunks = np.array([bvl.fixed_encode(x) for x in t], dtype=np.uint64)
    acc1 = chunks.sum(0)
    acc2 = chunks[rng.permutation(len(t))].sum(0)
    assert np.array_equal(acc1, acc2)
    exact = sum(_exact(x) for x in t)
    got = bvl.fixed_decode(acc1)
    assert got == float(Fraction(exact, 1 << 64))
    # split across "ranks" then summed: same bits
    parts = [chunks[:1234].sum(0), chunks[1234:4000].sum(0), chunks[4000:].sum(0)]
    assert bvl.fixed_decode(sum(parts)) == got
