#!/usr/bin/env python
"""Benchmark: block-Vecchia log-likelihood evaluations per second (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One "step" = one full ℓ(θ) evaluation (Alg. 1 l.10-30) of
the frozen plan — θ upload, gather, Matérn, joint factorisation, per-block
terms, exact reduction, (allreduce), ℓ back on the host — alternating two θ
values as an optimiser would.  Default workload: c4 (n = 1M, 3D, 50k blocks,
m = 100), the configuration BASELINE.json's metric is quoted on.  Under
torchrun each rank owns a cost-balanced contiguous range of blocks; one
ncclAllReduce per evaluation (strong scaling: the problem is fixed).

Timing: W warm-up steps; K timed steps bracketed by barrier + synchronize;
per step CUDA events on the library's own stream (torch.cuda.ExternalStream)
with an L2 flush (256 MiB memset) between steps outside the events; max over
ranks.  `e2e` repeats the measurement through bv_loglik_host_y (pinned host
y copied in, ℓ copied out, every step).  `cpu_baseline` times the CPU oracle
(test infrastructure) on a bounded sample on rank 0 at N = 1.
`--impl reference` times that oracle alone (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bvgen  # noqa: E402

FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # derived: SMs × FP64 FMA/clk × 2 × max clock (37.2)
METRIC = "block-Vecchia loglik evals/sec at n=1M (1/2/4/8 B200); FP64 TFLOP/s vs peak"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        time.sleep(0.15)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                pass

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def workload(cfg_name):
    c = bvgen.CONFIGS[cfg_name]
    return c


def matern_entries(plan, k_begin=0, k_end=None):
    """E = Σ N_k(N_k+1)/2 Matérn entries per evaluation (Σcon, Σcross, Σlk lower)."""
    l, m = plan.block_sizes()
    N = (l + m).astype(np.float64)[k_begin:k_end]
    return float(np.sum(N * (N + 1) / 2.0))


def algorithmic_flops(plan, k_begin=0, k_end=None):
    """F = Σ N_k³/3 over positions, N_k = m_k + l_k."""
    l, m = plan.block_sizes()
    N = (l + m).astype(np.float64)[k_begin:k_end]
    return float(np.sum(N ** 3 / 3.0))


def oracle_sample_time(plan, theta, target_s, reps=1):
    """Time the CPU oracle (Alg. 1 literal, FP64, all host cores) on a bounded
    leading range of positions sized for ~target_s; returns (evals/s, desc, seconds, cores)."""
    import oracle
    l, m = plan.block_sizes()
    N = (l + m).astype(np.float64)
    cost = N ** 3 / 3.0 + 40.0 * N * (N + 1) / 2
    cum = np.cumsum(cost) / cost.sum()
    # calibrate on ~0.5 % of the work
    k0 = int(np.searchsorted(cum, 0.005)) + 1
    t = time.perf_counter()
    oracle.bv_loglik(plan, theta, k_range=(0, k0), per_block=False)
    t1 = time.perf_counter() - t
    frac_target = min(1.0, target_s / max(1e-6, t1 / cum[k0 - 1]))
    k1 = max(k0, int(np.searchsorted(cum, frac_target)) + 1)
    k1 = min(k1, plan.bc)
    share = float(cum[k1 - 1])
    times = []
    for _ in range(reps):
        t = time.perf_counter()
        oracle.bv_loglik(plan, theta, k_range=(0, k1), per_block=False)
        times.append(time.perf_counter() - t)
    cores = os.cpu_count() or 1
    desc = (f"positions [0,{k1}) of {plan.bc} = {share * 100:.2f}% of the evaluation's cost "
            f"(N^3/3 + 40 E), scaled to one full evaluation")
    return [share / x for x in times], desc, times, cores


def run_reference(args):
    """The tier's reference arm: the CPU oracle (Alg. 1 literal, FP64, all host cores) as it stands,
    timed on the same workload — W untimed warm-up evaluations, then K timed ones.  Each step is one
    WHOLE evaluation when the oracle finishes one within ~8 s (c1-c4); above that (c5) a bounded
    leading sample of positions, scaled to one evaluation, is stated in `sample`."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    c = workload(args.config)
    plan = bvgen.cached_plan(args.config, m=args.m)
    theta = tuple(c["theta"])
    import oracle
    oracle.build()
    t = time.perf_counter()
    oracle.bv_loglik(plan, theta, per_block=False)
    first = time.perf_counter() - t
    whole = first <= 8.0
    cores = os.cpu_count() or 1
    if whole:
        for _ in range(max(0, args.warmup - 1)):
            oracle.bv_loglik(plan, theta, per_block=False)
        times = []
        for _ in range(max(1, args.steps)):
            t = time.perf_counter()
            oracle.bv_loglik(plan, theta, per_block=False)
            times.append(time.perf_counter() - t)
        per_eval_s = times
        desc = f"whole evaluations ({len(times)} timed after {max(1, args.warmup)} warm-up)"
    else:
        for _ in range(max(0, args.warmup - 1)):
            oracle_sample_time(plan, theta, target_s=2.0)
        rates, desc, times, cores = oracle_sample_time(plan, theta, target_s=2.0, reps=max(1, args.steps))
        per_eval_s = [1.0 / r for r in rates]
    value = len(per_eval_s) / sum(per_eval_s)
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * float(np.mean(per_eval_s)),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": config_block(args, c, plan),
           "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": "oracle", "sample": desc},
           "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def ablation_leg(args):
    """Run this script as a child with the ablation library; returns its mean kernel ms (or None)."""
    from paper_2410_04477_b200 import build as bvbuild
    try:
        libp = bvbuild.build_ablation()
        env = dict(os.environ, BV_LIB_PATH=libp)
        cmd = [sys.executable, os.path.abspath(__file__), "--ablation-child", "--config", args.config,
               "--steps", str(max(5, args.steps))] + (["--m", str(args.m)] if args.m else [])
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
        return float(json.loads(r.stdout.strip().splitlines()[-1])["kernel_ms"])
    except Exception as e:  # the ablation is a diagnostic: never fail the bench line
        print(f"ablation leg failed: {e!r}", file=sys.stderr)
        return None


def run_ablation_child(args):
    import torch
    import paper_2410_04477_b200 as bvl
    c = workload(args.config)
    plan = bvgen.cached_plan(args.config, m=args.m)
    theta = tuple(c["theta"])
    bv = bvl.BlockVecchia(plan, device=0)
    for _ in range(3):
        bv.loglik(theta)
    torch.cuda.synchronize()
    ks = []
    for _ in range(args.steps):
        bv.loglik(theta)
        ks.append(bv.last_kernel_ms())
    bv.close()
    print(json.dumps({"kernel_ms": float(np.mean(ks))}))
    return 0


def synth_gp_y(plan, theta, seed):
    """Exact zero-mean Matérn GRF draw at the plan's locations (c2 recipe: dense
    Cholesky of the n×n covariance, a generator step — torch FP64 on the GPU, not the product
    path).  Closed-form ν only."""
    import torch
    X = torch.from_numpy(plan.locs).cuda()
    r = torch.cdist(X, X, compute_mode="donot_use_mm_for_euclid_dist") / theta[1]
    nu = theta[2]
    poly = {0.5: 1.0, 1.5: 1.0 + r, 2.5: 1.0 + r + r * r / 3.0}[nu]
    S = theta[0] * poly * torch.exp(-r)
    del r
    Lc = torch.linalg.cholesky(S)
    del S
    eps = torch.from_numpy(bvgen.normal(seed, plan.n)).cuda()
    y = (Lc @ eps).cpu().numpy()
    del Lc
    torch.cuda.empty_cache()
    return y


def run_mle(args):
    """c2: one MLE fit: start (0.5, 0.1, 1.0), box [0.05,5]×[0.005,0.5]×[0.2,3],
    relative Δℓ < 1e-7 or 2000 evaluations; ν estimated, so nearly every evaluation takes the
    general-K_ν path.  value = evaluations per second over the whole fit (optimiser included)."""
    import torch
    import paper_2410_04477_b200 as bvl
    from paper_2410_04477_b200.mle import fit
    from paper_2410_04477_b200 import build as bvbuild
    args.config = "c2"
    torch.cuda.set_device(0)
    bvbuild.build()
    c = workload("c2")
    theta_true = tuple(c["theta"])
    plan = bvgen.cached_plan("c2")
    plan = plan.with_y(synth_gp_y(plan, theta_true, 100 * c["cfg"] + 2))
    bv = bvl.BlockVecchia(plan, device=0)
    for _ in range(3):
        bv.loglik(theta_true)
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        res = fit(bv.loglik)
    kern = bv.last_kernel_ms()
    bv.close()
    out = {"metric": "block-Vecchia MLE fit: loglik evals/sec over a full BOBYQA-style fit (c2)",
           "value": res["evals_per_s"], "unit": "evals/s", "n_gpus": 1, "steps": res["n_evals"], "warmup": 3,
           "ms_per_step": 1000.0 * res["wall_s"] / res["n_evals"], "higher_is_better": True, "scaling": "none",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (exact Matern GRF, dense Cholesky)",
           "config": dict(config_block(args, c, plan), workload="c2 MLE: n=20,000 2D, bc=500, m=60, "
                          "theta_true=(1.0, 0.052537, 1.5), start (0.5, 0.1, 1.0), nu estimated"),
           "mle": {"theta_hat": res["theta"], "loglik_hat": res["loglik"], "n_evals": res["n_evals"],
                   "wall_s": res["wall_s"], "converged": res["converged"], "theta_true": theta_true,
                   "last_kernel_ms": kern},
           "clocks": clk.summary()}
    if not args.no_cpu_baseline:
        import oracle
        oracle.build()
        t = time.perf_counter()
        ro = fit(lambda th: oracle.bv_loglik(plan, th, per_block=False)["loglik"])
        w = time.perf_counter() - t
        out["cpu_baseline"] = {"value": ro["n_evals"] / w, "unit": "evals/s", "cores": os.cpu_count() or 1,
                               "kind": "oracle", "sample": "the same full MLE fit on the CPU oracle",
                               "theta_hat": ro["theta"], "n_evals": ro["n_evals"], "seconds": w}
    print(json.dumps(out))
    return 0


def run_predict(args):
    """Alg. 2 at the config's scale: n* = n/10 new locations (same
    distribution), bc* = bc/10 prediction blocks, the config's m.  value = predicted points per
    second (mean + variance + block covariances), device-timed around bv_predict (host marshalling
    of the prediction plan included — the paper predicts once per fit)."""
    import torch
    import paper_2410_04477_b200 as bvl
    from paper_2410_04477_b200 import build as bvbuild
    torch.cuda.set_device(0)
    bvbuild.build()
    c = workload(args.config)
    plan = bvgen.cached_plan(args.config, m=args.m)
    n_new, bc_new = max(1, plan.n // 10), max(1, plan.bc // 10)
    new = bvgen.locations(c["cfg"] + 50, n_new, plan.d)
    pp = bvgen.make_pred_plan(plan.locs, new, bc_new, plan.m)
    theta = tuple(c["theta"])
    bv = bvl.BlockVecchia(plan, device=0)
    for _ in range(max(1, args.warmup)):
        bv.predict(theta, pp)
    torch.cuda.synchronize()
    ts, kms = [], []
    for _ in range(args.steps):
        t = time.perf_counter()
        bv.predict(theta, pp, want_cov=True)
        ts.append(time.perf_counter() - t)
        kms.append(bv.last_kernel_ms())  # events around the prediction kernel alone
    bv.close()
    lsz = np.bincount(pp.block_id, minlength=bc_new)
    N = (lsz + plan.m).astype(np.float64)
    flops = float(np.sum((plan.m ** 3) / 3.0 + plan.m ** 2 * lsz + plan.m * lsz * lsz))  # m eliminated columns
    sec = float(np.median(ts))
    out = {"metric": "block-Vecchia prediction (Alg. 2): predicted points/sec", "value": n_new / sec,
           "unit": "points/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * sec,
           "higher_is_better": True, "scaling": "none", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{args.config} prediction: n*={n_new:,} new points, bc*={bc_new:,} blocks, "
                                  f"m={plan.m}, theta={theta}", "n_train": plan.n, "n_new": n_new, "bc_new": bc_new,
                      "m": plan.m, "max_joint": int(N.max())},
           "fp64_tflops": flops / sec / 1e12, "note": "wall time of bv_predict incl. host-side plan marshalling",
           "kernel": {"ms": float(np.median(kms)), "points_per_s": n_new / (float(np.median(kms)) / 1e3),
                      "fp64_tflops": flops / (float(np.median(kms)) / 1e3) / 1e12,
                      "what": "CUDA events around the prediction kernel (bv_last_kernel_ms after bv_predict)"}}
    print(json.dumps(out))
    return 0


def config_block(args, c, plan):
    return {"workload": f"{args.config}: n={plan.n:,} {plan.d}D, bc={plan.bc:,} K-means blocks, m={plan.m}, "
                        f"random ordering, Matern theta={tuple(c['theta'])}",
            "n": plan.n, "d": plan.d, "bc": plan.bc, "m": plan.m, "theta": list(c["theta"]),
            "l2": "flushed between steps (256 MiB memset outside the timed events)",
            "parallelism": f"blocks partitioned over {args.gpus} GPU(s), 1 allreduce/eval"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)  # ≥ 1 s of timed evaluations at c4
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(bvgen.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--m", type=int, default=None, help="override the config's m (c5 sweep: 30/60/120/200)")
    ap.add_argument("--no-ablation", action="store_true", help="skip the factorisation-only ablation leg")
    ap.add_argument("--ablation-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--mle", action="store_true", help="c2 workload: a full MLE fit (hundreds of evaluations)")
    ap.add_argument("--predict", action="store_true",
                    help="Alg. 2 block prediction on the config's plan (new points = n/10, blocks = bc/10)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.ablation_child:
        return run_ablation_child(args)
    if args.mle:
        return run_mle(args)
    if args.predict:
        return run_predict(args)

    import torch
    import paper_2410_04477_b200 as bvl
    from paper_2410_04477_b200 import build as bvbuild

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        bvbuild.build()
    if dist:
        dist.barrier()
    c = workload(args.config)
    plan = bvgen.cached_plan(args.config, m=args.m) if rank == 0 else None
    if dist:
        dist.barrier()
        if rank != 0:
            plan = bvgen.cached_plan(args.config, m=args.m)
    theta_a = tuple(c["theta"])
    theta_b = (theta_a[0] * 1.05, theta_a[1] * 0.97, theta_a[2])
    nid = None
    if world > 1:
        obj = [bvl.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    bv = bvl.BlockVecchia(plan, device=local, rank=rank, world=world, nccl_id=nid)
    F_local = algorithmic_flops(plan, bv.k_begin, bv.k_end)
    F_total = algorithmic_flops(plan)
    ext = torch.cuda.ExternalStream(bv.stream_ptr, device=torch.device("cuda", local))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timed_loop(fn, K):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        kern = []
        for i in range(K):
            with torch.cuda.stream(ext):
                flush.zero_()
                ev[i][0].record(ext)
            fn(theta_a if i % 2 == 0 else theta_b)
            ev[i][1].record(ext)
            kern.append(bv.last_kernel_ms())
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in ev], kern

    for i in range(max(3, args.warmup)):
        bv.loglik(theta_a if i % 2 == 0 else theta_b)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        step_ms, kern_ms = timed_loop(bv.loglik, args.steps)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = float(sum(step_ms))
    kmean = float(np.mean(kern_ms))

    # e2e through the host-buffer C-ABI call
    y_host = torch.from_numpy(np.ascontiguousarray(plan.y)).pin_memory()
    for i in range(2):
        bv.loglik_host_y(y_host, theta_a)
    if dist:
        dist.barrier()
    e2e_ms, _ = timed_loop(lambda th: bv.loglik_host_y(y_host, th), args.steps)
    e2e_total = float(sum(e2e_ms))

    def max_all(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    total_ms = max_all(total_ms)
    e2e_total = max_all(e2e_total)
    kmean_max = max_all(kmean)
    value = args.steps / (total_ms / 1000.0)
    e2e_value = args.steps / (e2e_total / 1000.0)
    achieved = F_local / (kmean / 1000.0) / 1e12
    roofline = {"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None,
                "kernel": "block kernels (all size buckets: bv_block_v3 CTA kernel, bv_block_w warp kernel; gather + "
                          "Matern + joint Cholesky + terms + exact reduction)",
                "kernel_ms": kmean, "flops_per_launch": F_local,
                "peak_source": "derived FP64: 148 SM x 64 FMA/clk x 2 x 1.965 GHz; DMMA probe measured 37.13 "
                               "(tools/peaks)"}
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):  # DRAM bytes (read+write) of the block kernels per evaluation, from ncu --set full
        try:
            tr = json.load(open(prof)).get(args.config)
            if tr:
                roofline["traffic"] = tr["dram_bytes_per_eval_est"]
                roofline["traffic_source"] = tr["source"]
        except Exception:
            pass
    E_local = matern_entries(plan, bv.k_begin, bv.k_end)
    matern = {"entries_per_eval": E_local, "entries_per_s": E_local / (kmean / 1000.0),
              "what": "SURVEY 8d (iii): Matern entries E = sum N(N+1)/2 per evaluation over the block-kernel time"}
    fp64x = None
    pf = os.path.join(ROOT, "profiles", "ncu_fp64_r02.json")
    if os.path.exists(pf):  # executed FP64 work of one evaluation, from ncu instruction counters
        try:
            rec = json.load(open(pf)).get(args.config if args.m is None else f"{args.config}_m{args.m}")
            if rec:
                fx = rec["fp64_flops_executed_per_eval"]
                fp64x = {"flops_executed_per_eval": fx, "executed_over_algorithmic": fx / F_total,
                         "achieved_executed_tflops": fx / (kmean / 1000.0) / 1e12,
                         "frac_executed": fx / (kmean / 1000.0) / 1e12 / FP64_PEAK_TFLOPS,
                         "formula": rec["formula"], "source": rec["source"]}
        except Exception:
            pass
    out = {"metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
           "warmup": max(3, args.warmup), "ms_per_step": total_ms / args.steps, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": config_block(args, c, plan),
           "fp64_tflops_whole_eval": F_total / (total_ms / args.steps / 1000.0) / 1e12,
           "roofline": roofline, "matern": matern,
           "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": int(8 * plan.n + 192),
                   "d2h_bytes_per_step": 64},
           "gpu_launches": int(bv.launches_per_eval * args.steps),
           "clocks": clk.summary()}
    if fp64x:
        out["fp64_executed"] = fp64x
    if rank == 0 and world == 1 and not args.no_ablation:
        ab = ablation_leg(args)
        if ab is not None:
            out["factorization_only"] = {
                "what": "SURVEY 8d (v): the same block kernels with the Matern fill replaced by a cheap SPD fill "
                        "(libbv_fill.so, -DBV_ABL_FILL); F / kernel time = FP64 factorisation rate",
                "kernel_ms": ab, "achieved": F_local / (ab / 1000.0) / 1e12, "unit": "TFLOP/s",
                "frac": F_local / (ab / 1000.0) / 1e12 / FP64_PEAK_TFLOPS,
                "generation_ms_est": kmean - ab}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rates, desc, times, cores = oracle_sample_time(plan, theta_a, target_s=15.0)
        out["cpu_baseline"] = {"value": rates[0], "unit": "evals/s", "cores": cores, "kind": "oracle",
                               "sample": desc, "seconds": times[0]}
    if rank == 0:
        print(json.dumps(out))
    bv.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
