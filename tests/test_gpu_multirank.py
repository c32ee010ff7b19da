"""The world > 1 device layout on one GPU (-m gpu), rank by rank.

Blocks are independent given θ, so a rank's evaluation needs
nothing from the other ranks until the one final sum.  bv_setup_rank_local
builds exactly the layout rank r of G gets under NCCL (its contiguous,
cost-balanced position range, the rank-local neighbour slice with rebased
offsets) without a communicator; the G handles run one after another on
cuda:0 (no rank waits on another).  Checked against the single-rank handle:
  * the G partial fixed-point accumulators sum (as integers) to the single-rank
    accumulator, so ℓ is bitwise the same;
  * every rank's d_k, u_k equal the global ones on its range, bitwise;
  * a non-PD failure is reported by the owning rank at its GLOBAL position.
"""
import numpy as np
import pytest

import bvgen
import oracle
import paper_2410_04477_b200 as bvl
from paper_2410_04477_b200 import BlockVecchia, NotPositiveDefinite

pytestmark = pytest.mark.gpu


def _plan(case):
    theta = (1.0, 0.052537, 1.5)
    if case == "c2":
        p = bvgen.cached_plan("c2")
    else:  # a c4-shaped slice: 3D, 17 layers, m = 100
        p = bvgen.make_plan("c4", n=100_000, bc=5_000, m=100, cfg=4)
    return p.with_y(oracle.simulate_bv(p, theta, bvgen.normal(7001, p.n))), theta


@pytest.mark.parametrize("case", ["c2", "c4slice"])
def test_rank_local_partition_sums_bitwise(case):
    p, theta = _plan(case)
    one = BlockVecchia(p)
    acc1 = one.loglik_acc(theta)
    ll1, d1, u1 = one.loglik_terms(theta)
    one.close()
    assert bvl.fixed_decode(acc1[:6]) == ll1
    for G in (2, 4, 8):
        tot = np.zeros(6, dtype=np.uint64)
        prev_end = 0
        for r in range(G):
            h = BlockVecchia(p, rank=r, world=G, rank_local=True)
            assert h.k_begin == prev_end
            prev_end = h.k_end
            acc = h.loglik_acc(theta)
            assert acc[6] == 0 and acc[7] == np.uint64(2**64 - 1)
            tot += acc[:6]  # integer chunk sums: what the one ncclAllReduce adds
            _, d, u = h.loglik_terms(theta)
            h.close()
            assert np.array_equal(d, d1[h.k_begin:h.k_end]) and np.array_equal(u, u1[h.k_begin:h.k_end])
        assert prev_end == p.bc
        assert np.array_equal(tot, acc1[:6]), (G, tot, acc1[:6])
        assert bvl.fixed_decode(tot) == ll1  # bitwise, for every G


def test_rank_local_failure_has_global_position():
    theta = (1.0, 0.1, 0.5)
    p = bvgen.make_plan("c1", n=4000, bc=80, m=30, cfg=71)
    cuts = bvl.partition(*p.block_sizes(), 4)
    k_bad = int(cuts[2]) + 5  # inside rank 2's range
    locs = p.locs.copy()
    mem = np.where(p.block_id == p.order[k_bad])[0]
    locs[mem[1]] = locs[mem[0]]
    q = bvgen.Plan(locs, bvgen.normal(7102, p.n), p.block_id, p.order, p.nbr_ptr, p.nbr_idx)
    with pytest.raises(NotPositiveDefinite) as e:
        BlockVecchia(q).loglik(theta)
    assert e.value.failed_position == k_bad
    for r in range(4):
        h = BlockVecchia(q, rank=r, world=4, rank_local=True)
        if r == 2:
            with pytest.raises(NotPositiveDefinite) as e:
                h.loglik(theta)
            assert e.value.failed_position == k_bad  # global k, not the rank-local index
            acc = h.loglik_acc(theta)
            assert int(acc[6]) == 1 and int(acc[7]) >> 8 == k_bad
        else:
            h.loglik(theta)
        h.close()
