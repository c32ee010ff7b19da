"""Multi-rank host logic on CPU (-m "not gpu"): world_size 2 over gloo.

The GPU path splits positions into contiguous cost-balanced ranges
(bv_partition), each rank adds its blocks' exact fixed-point terms
(bv_fixed_encode, chunk sums), and ONE allreduce(sum) of the 7 uint64 slots
combines them.  Here the per-block terms come from the CPU
oracle; the test checks that the two-rank result is bitwise the single-rank
result and that a failure count/min position travel the same way.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bvgen
import oracle
import paper_2410_04477_b200 as bvl
from paper_2410_04477_b200 import build as bvbuild


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _acc_for_range(t, k0, k1):
    acc = np.zeros(7, dtype=np.uint64)
    for x in t[k0:k1]:
        acc[:6] += bvl.fixed_encode(float(x)).astype(np.uint64)
    return acc


def _worker(rank, world, port, t, l, m, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cuts = bvl.partition(l, m, world)
    k0, k1 = int(cuts[rank]), int(cuts[rank + 1])
    acc = _acc_for_range(t, k0, k1)
    acc[6] = 1 if (rank == 1) else 0  # one rank reports a failed block
    ten = torch.from_numpy(acc.view(np.int64).copy())
    dist.all_reduce(ten, op=dist.ReduceOp.SUM)  # the one collective per evaluation
    fail_pos = torch.tensor([k0 + 3 if rank == 1 else 2**62], dtype=torch.int64)
    if int(ten[6]) > 0:  # off the hot path: the smallest failing position
        dist.all_reduce(fail_pos, op=dist.ReduceOp.MIN)
    tot = ten.numpy().view(np.uint64)
    out[rank] = (bvl.fixed_decode(tot[:6]), int(tot[6]), int(fail_pos[0]), (k0, k1))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_exact_sum_matches_single_rank(world):
    bvbuild.build()
    theta = (1.0, 0.052537, 1.5)
    p = bvgen.make_plan("c1", n=3000, bc=60, m=30, cfg=51)
    p = p.with_y(oracle.simulate_bv(p, theta, bvgen.normal(5102, p.n)))
    r = oracle.bv_loglik(p, theta)
    l, m = p.block_sizes()
    single = bvl.fixed_decode(_acc_for_range(r["t"], 0, p.bc)[:6])
    assert abs(single - r["loglik"]) <= 1e-12 * abs(r["loglik"])
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, r["t"], l, m, out), nprocs=world, join=True)
    vals = [out[k] for k in range(world)]
    for v, cnt, fp, rng in vals:
        assert v == single  # bitwise, on every rank
        assert cnt == 1
    ranges = [v[3] for v in vals]
    assert ranges[0][0] == 0 and ranges[-1][1] == p.bc
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    assert vals[0][2] == ranges[1][0] + 3
