#!/usr/bin/env python
"""Benchmark of the MRA log-likelihood hot path on B200 (BASELINE.json metric:
observations/sec per MRA log-lik evaluation, fp64, and the fraction of the fp64 roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl mra|reference]

One step = one full MRA log-likelihood evaluation (prior pass + posterior pass, every §8(a)
row) of the config's synthetic data for a fixed plan, y already resident in HBM (the paper's
"excluding loading the data and building the structure"). N > 1 ranks (one
process per GPU: torchrun, or spawned by this script when --gpus N is given without WORLD_SIZE)
shard the subtrees; each plan holds its own NCCL communicator (opts.nccl_id) and
mra_loglik_dev runs the exchange step inside the library (broadcast of the above-shard prior rows,
reduce of the packed shard outputs to rank 0, broadcast of log L); time = max over ranks (CUDA
events). The headline value is timed with the library's per-launch profiling OFF; kernel times and
the roofline come from a separate profiled pass of the same steps.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "observations/sec per MRA log-lik eval (fp64)"
UNIT = "obs/s"
DEFAULT_CONFIG = "C3"
# fp64 roofline denominator: MEASURED_PEAKS.json bf16 x the guide's nominal fp64-tensor:bf16 ratio
# (blackwell_cuda_programming.md: B200 FP64 tensor 45 TFLOPS vs 2.25 PFLOPS dense bf16)
FP64_NOMINAL_TF = 45.0
BF16_NOMINAL_TF = 2250.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ flop model (§8(d))
def leaf_flops(n, P, r):
    """SURVEY.md §8(d) algorithmic flops of one leaf with n observations, P = M-1 ancestor levels."""
    n = np.asarray(n, dtype=np.float64)
    Pr = P * r
    f = P * P * n * r * r                      # W chain + V triangular solves
    f += n * (n + 1) * Pr                      # Sigma_j = C - V V^T (symmetric, half)
    f += n ** 3 / 3.0                          # Cholesky
    f += n * n * (Pr + 1)                      # G = L^{-1} [V | y]
    f += Pr * (Pr + 1) * n                     # A = G^T G (symmetric, half)
    f += 2 * Pr * n + 2 * n                    # omega, u
    return np.where(n > 0, f, 0.0)


def interior_flops(m, r):
    """prior + merge flops of one level-m region."""
    prior = m * (m - 1) * r ** 3 + (m - 1) * r ** 3 + r ** 3 / 3.0
    merge = r ** 3 / 3.0 + r * r * ((m - 1) * r + 1) + (m - 1) * r * ((m - 1) * r + 1) * r + 2 * (m - 1) * r * r
    return prior, merge


def class_flops(leaf_sizes, M, J, r):
    """§8(d) algorithmic flops per evaluation split by the kernel classes of mra_kernel_times."""
    n = np.asarray(leaf_sizes, dtype=np.float64)
    n = n[n > 0]
    P = M - 1
    Pr = P * r
    # leaves with n <= ncol are solved through the explicit inverse by k_wide_trsm ("solve"); larger leaves
    # by the blocked substitution interleaved with their factorization ("factor"), DESIGN.md §5
    xm = n <= Pr + 1
    out = {"chain": float(np.sum(P * P * n * r * r)), "sigma": float(np.sum(n * (n + 1) * Pr)),
           "factor": float(np.sum(n ** 3 / 3.0) + np.sum((n * n * (Pr + 1))[~xm])),
           "solve": float(np.sum((n * n * (Pr + 1))[xm])),
           "syrk_merge": float(np.sum(Pr * (Pr + 1) * n + 2 * Pr * n + 2 * n))}
    prior = merge = 0.0
    for m in range(1, M):
        p_, g_ = interior_flops(m, r)
        prior += J ** (m - 1) * p_
        if m == M - 1:
            out["syrk_merge"] += J ** (m - 1) * g_
        else:
            merge += J ** (m - 1) * g_
    out["prior"], out["merge"] = prior, merge
    out["bottom"] = sum(out[k] for k in ("chain", "sigma", "factor", "solve", "syrk_merge"))
    return out


KERNEL_NAMES = {"prior": "k_prior (levels 1..M-1 W chains, Cholesky, inverse)",
                "bottom": "k_bottom (one CTA per level-(M-1) region: leaves + level M-1 merge)",
                "merge": "k_merge (levels M-2..1)",
                "chain": "k_wide_chain (leaf V chains: m single-segment GEMMs over the covariance blocks in place)",
                "sigma": "k_wide_sigma (Sigma_j = C(S,S) + tau2 I - V V^T tiles)",
                "factor": "k_wide_update/diag/panel_x (blocked Cholesky of Sigma_j, X = L^{-1})",
                "solve": "k_wide_trsm (G = X [V | y])",
                "syrk_merge": "k_wide_mtile (Atilde = G^T G tiles + level M-1 merge dataflow)"}


def flop_model(leaf_sizes, M, J, r):
    P = M - 1
    leaves = float(np.sum(leaf_flops(leaf_sizes, P, r)))
    prior = merge = merge_bottom = 0.0
    for m in range(1, M):
        p, g = interior_flops(m, r)
        prior += J ** (m - 1) * p
        merge += J ** (m - 1) * g
        if m == M - 1:
            merge_bottom = J ** (m - 1) * g
    return dict(total=leaves + prior + merge, leaves=leaves, prior=prior, merge=merge,
                bottom=leaves + merge_bottom)


# --------------------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region, plus one NVML
    sample at its start and one at its end (regions shorter than the sampling period still get samples)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None
        self.extra = []   # NVML samples at start / stop: a timed region shorter than nvidia-smi's period

    def _nvml_sample(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            names = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                     "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                     "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                     "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self.extra.append((sm, mx, {k for k, bit in names.items() if r & bit}))
        except Exception:
            pass

    def start(self):
        self.extra = []
        self._nvml_sample()
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        self._nvml_sample()
        out = ""
        if self.p is not None:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
                out = ""
        sm, mx, reasons = [], 0.0, set()
        for s_, m_, r_ in self.extra:
            sm.append(s_)
            mx = max(mx, m_)
            reasons |= r_
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nme, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nme)
        if not sm:
            return None
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return pk, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def measured_fp64_peak():
    """Best DMMA TFLOP/s line of the committed fp64 microbenchmark output (profiles/fp64_peak_r01.txt)."""
    try:
        best = 0.0
        for line in open(os.path.join(ROOT, "profiles", "fp64_peak_r01.txt")):
            if line.startswith("DMMA"):
                best = max(best, float(line.split(":")[-1].split()[0]))
        return best or None
    except Exception:
        return None


def region_box(x, y, J, level, t):
    """Box of region (level, t) by the paper's split rule (only used to pre-select the oracle's
    timing sample; the oracle assigns the points itself)."""
    x0, x1, y0, y1 = x.min(), x.max(), y.min(), y.max()
    b = [x0, x1 + 0.01 * (x1 - x0), y0, y1 + 0.01 * (y1 - y0)]
    path = []
    for _ in range(level - 1):
        path.append(t % J)
        t //= J
    for c in reversed(path):
        mx, my = 0.5 * (b[0] + b[1]), 0.5 * (b[2] + b[3])
        if J == 4:
            b = [mx, b[1], b[2], b[3]] if c & 1 else [b[0], mx, b[2], b[3]]
            b = [b[0], b[1], my, b[3]] if c & 2 else [b[0], b[1], b[2], my]
        elif (b[1] - b[0]) >= (b[3] - b[2]):
            b = [mx, b[1], b[2], b[3]] if c else [b[0], mx, b[2], b[3]]
        else:
            b = [b[0], b[1], my, b[3]] if c else [b[0], b[1], b[2], my]
    return b


def oracle_sample(w, theta, budget_s, seed=0, max_samples=64):
    """Time the CPU oracle (as it stands) on a bounded sample of the same workload: whole subtrees
    rooted at level max(1, M-3) (<= 64 leaves each), evaluated with the oracle's subtree mode on the
    subtree's points plus the 4 bounding-box extremes (so the oracle builds the identical tree).
    Returns (obs/s, obs, seconds, samples, threads)."""
    import oracle
    lvl = max(1, w.M - 3)
    nreg = w.J ** (lvl - 1)
    rng = np.random.default_rng(seed)
    ext = np.unique([np.argmin(w.x), np.argmax(w.x), np.argmin(w.y), np.argmax(w.y)])
    tot_obs, tot_s, k = 0, 0.0, 0
    while (tot_s < budget_s or k == 0) and k < max_samples:
        t = int(rng.integers(0, nreg))
        b = region_box(w.x, w.y, w.J, lvl, t)
        sel = np.nonzero((w.x >= b[0]) & (w.x < b[1]) & (w.y >= b[2]) & (w.y < b[3]))[0]
        idx = np.union1d(sel, ext)
        xs, ys, zs = w.x[idx], w.y[idx], w.z[idx]
        t0 = time.perf_counter()
        oracle.run(xs, ys, zs, w.M, w.J, w.r, theta, target=(lvl, t))
        tot_s += time.perf_counter() - t0
        tot_obs += sel.size
        k += 1
    return tot_obs / tot_s, tot_obs, tot_s, k, oracle.threads(), lvl


# ------------------------------------------------------------------------- arms
def cpu_info():
    """CPU model and core count of the host the oracle baseline ran on."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def run_reference(args, rank):
    """--impl reference: the oracle (the deliberately slow CPU baseline) on the box's host cores."""
    if rank != 0:
        return
    w = synth.make(args.config, n=args.n)
    theta = w.thetas[0]
    import oracle
    oracle.build()
    budget = args.ref_budget
    for _ in range(args.warmup):
        oracle_sample(w, theta, 0.0, seed=123, max_samples=1)
    vals, obs, secs, samples = [], 0, 0.0, 0
    for s in range(args.steps):
        v, o, sec, k, thr, lvl = oracle_sample(w, theta, budget, seed=s)
        vals.append(v); obs += o; secs += sec; samples += k
    value = obs / secs
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": config_block(w, None, args.gpus),
            "cpu_baseline": dict({"value": value, "unit": UNIT, "cores": thr, "kind": "oracle",
                                  "sample": f"{samples} whole level-{lvl} subtrees ({obs} obs) of {w.name}, "
                                            f"oracle subtree mode, {secs:.1f} s CPU wall"}, **cpu_info()),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_block(w, plan, ngpu):
    th = w.thetas[0]
    c = {"workload": f"{w.name}: n={w.n:,} {w.recipe}; M={w.M} J={w.J} r={w.r}"
                     + (f" (r_hat={plan.r_hat})" if plan else ""),
         "n_obs": w.n, "M": w.M, "J": w.J, "r": w.r,
         "theta": {"cov": ["exponential", "matern32"][th[0]], "sigma2": th[1], "rho": th[2], "tau2": th[3]},
         "parallelism": f"subtree-shard x{ngpu}" if ngpu > 1 else "1 GPU",
         "l2": "inputs larger than L2 (plan + prior state >> 126 MB) and L2 flushed between steps"}
    return c


def run_gpu(args, rank, world, local_rank):
    import torch
    import paper_1905_00141_b200 as mra
    from paper_1905_00141_b200 import build as mbuild
    if rank == 0:
        mbuild.build()
    if world > 1:
        torch.distributed.barrier()
    mra.load_library()
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    t0 = time.time()
    w = synth.make(args.config, n=args.n, device=dev)
    if args.M:
        w.M = args.M
    log(f"[rank {rank}] data {w.name} n={w.n} in {time.time() - t0:.1f}s")
    t0 = time.time()
    lanes = args.theta_lanes if args.theta_lanes is not None else 1
    nccl_id = None
    if world > 1:   # rank 0 makes the id of the plan's own communicator; every rank receives it
        obj = [mra.mra_nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    plan = mra.mra_plan_create(w.x, w.y, w.M, w.J, w.r, device=local_rank, stream=stream, rank=rank,
                               world=world, stream_prior=args.stream_prior, theta_lanes=lanes, nccl_id=nccl_id,
                               graph=bool(args.graph))
    torch.cuda.synchronize()
    plan_s = time.time() - t0
    log(f"[rank {rank}] plan in {plan_s:.1f}s: n_retained={plan.n_retained} r_hat={plan.r_hat}")
    thetas = w.thetas if args.config == "C4" else w.thetas[:1]
    zd = torch.from_numpy(w.z).to(dev)
    zpin = torch.from_numpy(w.z).pin_memory()
    zpin_np = zpin.numpy()
    flush = torch.empty(256 * 1024 * 1024 // 8 * 2, dtype=torch.float64, device=dev)   # 256 MB > L2

    def step(host=False):
        # the public API a user calls: every rank gets log L (the exchange runs inside the library at N > 1)
        if len(thetas) > 1:   # a sweep: the batch entry points (theta lanes run concurrently)
            if host:
                return list(mra.mra_loglik_batch(plan, zpin_np, thetas))
            return list(mra.mra_loglik_batch_dev(plan, zd, thetas))
        if host:
            return [mra.mra_loglik(plan, zpin_np, thetas[0])["loglik"]]
        return [mra.mra_loglik_dev(plan, zd, thetas[0])["loglik"]]

    def timed(n, host=False, prof=False):
        ev = []
        launches = 0
        if prof:
            mra.mra_profile(plan, True)
        sampler = ClockSampler(local_rank)
        sampler.start()
        for _ in range(n):
            flush.fill_(1.0)
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            lls = step(host)
            b.record(stream)
            torch.cuda.synchronize()
            ev.append(a.elapsed_time(b))
            launches += mra.mra_last_launches(plan)
        clocks = sampler.stop()
        ms = float(np.sum(ev))
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        kt = None
        if prof:
            t = mra.mra_kernel_times(plan)
            mra.mra_profile(plan, False)
            kt = ([t[k][0] for k in mra.KERNEL_CLASSES], [t[k][1] for k in mra.KERNEL_CLASSES])
        timed.last_steps = list(ev)   # per-step device ms of this rank (mean(sd), median)
        return ms, lls, launches, clocks, kt

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # headline: library profiling off (no per-launch events inside the timed region)
    ms, lls, launches, clocks, _ = timed(args.steps)
    step_list = list(timed.last_steps)
    e2e_steps = max(1, min(args.steps, 3))
    ms_e2e, _, _, _, _ = timed(e2e_steps, host=True)
    # kernel classes and the roofline: a separate pass of the same steps with per-launch CUDA events
    prof_ms, _, _, _, kt = timed(args.steps, prof=True)
    if rank != 0:
        return
    ntheta = len(thetas)
    N = plan.n_retained
    per_step = ms / args.steps
    value = N * ntheta / (per_step / 1e3)
    e2e_val = N * ntheta / ((ms_e2e / e2e_steps) / 1e3)
    # roofline of the dominant kernel (bottom: leaves + level M-1 merge)
    lay = mra.mra_plan_layout(plan)
    sizes = np.diff(lay["leaf_off"])
    fm = flop_model(sizes, w.M, w.J, plan.r_hat)
    pk, src = peaks()
    bf16 = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    derived64 = bf16 * FP64_NOMINAL_TF / BF16_NOMINAL_TF
    meas64 = measured_fp64_peak()
    peak64 = meas64 or derived64
    steps_th = args.steps * ntheta
    cf = class_flops(sizes, w.M, w.J, plan.r_hat)
    # covariance generation is a write stream: 8 B per generated entry, n_j x (P r_hat + 1) per leaf
    covgen_bytes = float(np.sum(sizes)) * ((w.M - 1) * plan.r_hat + 1) * 8.0
    kms = dict(zip(mra.KERNEL_CLASSES, kt[0]))
    kcnt = dict(zip(mra.KERNEL_CLASSES, kt[1]))
    names = dict(KERNEL_NAMES)
    if kcnt.get("chain") and not kcnt.get("sigma"):
        # the chains and Sigma tiles ran as one dataflow kernel (k_wide_chsig), timed as the chain class
        cf = dict(cf, chain=cf["chain"] + cf["sigma"])
        names["chain"] = "k_wide_chsig (leaf V chains + Sigma_j tiles as one dataflow)"
    roof = None
    cand = [k for k in KERNEL_NAMES if kcnt.get(k)]
    if cand:
        dom = max(cand, key=lambda k: kms[k])   # the dominant kernel class of the step
        launch_ms = kms[dom] / kcnt[dom]
        flops_launch = cf[dom] / (kcnt[dom] / steps_th)
        achieved = flops_launch / (launch_ms / 1e3) / 1e12
        traffic = None
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
            ent = tj.get(w.name, {})
            if ent.get("class") == dom:
                traffic = ent.get("bytes_per_launch")
        except Exception:
            pass
        roof = {"bound": "tensor", "achieved": round(achieved, 3), "peak": round(peak64, 3), "unit": "TFLOP/s",
                "frac": round(achieved / peak64, 4), "traffic": traffic, "kernel": names[dom],
                "class": dom, "flops_per_launch": flops_launch, "launch_ms": launch_ms,
                "peak_source": (f"measured fp64 DMMA peak of this B200 pool (profiles/fp64_peak_r01.txt, "
                                f"tools/fp64_peak.cu); the guide-derived figure {src} bf16_tflops_sustained "
                                f"{bf16} x {FP64_NOMINAL_TF}/{BF16_NOMINAL_TF} = {derived64:.2f} is lower")
                               if meas64 else f"{src} bf16_tflops_sustained {bf16} x {FP64_NOMINAL_TF}/{BF16_NOMINAL_TF}",
                "kernel_share_of_step": round(kms[dom] / prof_ms, 4),
                "profiled_pass_ms_per_step": round(prof_ms / args.steps, 3),
                "per_class_tflops": {k: round(cf[k] * steps_th / (kms[k] / 1e3) / 1e12, 2) for k in cand},
                "covgen": ({"kernel": "k_wide_covfill (covariance blocks of the leaf chains, HBM writes)",
                            "ms_per_step": round(kms["covgen"] / steps_th, 3),
                            "achieved_gbs": round(covgen_bytes * steps_th / (kms["covgen"] / 1e3) / 1e9, 1),
                            "hbm_peak_gbs": pk.get("hbm_gbs"),
                            "bytes_per_step": covgen_bytes}
                           if kcnt.get("covgen") else None),
                "step_fp64_tflops": round(fm["total"] * steps_th / (ms / 1e3) / 1e12, 3),
                "step_frac_of_peak": round(fm["total"] * steps_th / (ms / 1e3) / 1e12 / peak64, 4)}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, o, sec, k, thr, lvl = oracle_sample(w, thetas[0], args.cpu_budget)
        cpu = dict({"value": v, "unit": UNIT, "cores": thr, "kind": "oracle",
                    "sample": f"{k} whole level-{lvl} subtrees ({o} obs) of {w.name}, oracle subtree mode, "
                              f"{sec:.1f} s CPU wall"}, **cpu_info())
    pred = None
    if world == 1 and args.predict > 0:
        # NEXT-1: posterior mean / variance of X at random locations of the domain
        rng = np.random.default_rng(7)
        qx = rng.uniform(float(np.min(w.x)), float(np.max(w.x)), args.predict)
        qy = rng.uniform(float(np.min(w.y)), float(np.max(w.y)), args.predict)
        mra.mra_loglik(plan, zpin_np, thetas[0], posterior=True)
        mra.mra_predict(plan, qx[:1000], qy[:1000])          # warm-up (workspace allocation)
        ts = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pm, pv = mra.mra_predict(plan, qx, qy)
            ts.append(time.perf_counter() - t0)
        tp_ = min(ts)
        pred = {"queries": args.predict, "value": args.predict / tp_, "unit": "queries/s", "seconds": tp_,
                "what": "mra_predict (host query arrays in, host mean/var out; leaf assignment + sort on the "
                        "host, one k_predict launch) after a posterior-state evaluation of the same data",
                "finite": int(np.sum(np.isfinite(pm))), "var_min": float(np.nanmin(pv))}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config_block(w, plan, world), theta_lanes=lanes, cuda_graph=bool(args.graph)),
            "loglik": lls[0], "n_theta_per_step": ntheta, "flops_per_step": fm["total"] * ntheta,
            "e2e": {"value": e2e_val, "unit": UNIT,
                    # a sweep (mra_loglik_batch) copies y once per step, single evaluations once per theta
                    "h2d_bytes_per_step": 8 * w.n,
                    "d2h_bytes_per_step": 8 * ntheta},
            "step_ms": {"mean": float(np.mean(step_list)), "sd": float(np.std(step_list, ddof=1)) if len(step_list) > 1
                        else 0.0, "median": float(np.median(step_list)), "runs": len(step_list),
                        "note": "rank 0's per-step device times; ms_per_step is the max over ranks of their sums / steps"},
            "gpu_launches": int(launches),
            "kernel_ms": {k: round(kms[k], 3) for k in mra.KERNEL_CLASSES},
            "kernel_launches": {k: int(kcnt[k]) for k in mra.KERNEL_CLASSES},
            "roofline": roof, "cpu_baseline": cpu, "clocks": clocks}
    line["plan_memory"] = mra.mra_plan_memory(plan)   # streamed prior rows (NEXT-4), chunking, device bytes
    line["plan_seconds"] = round(plan_s, 3)   # S0 (device build, not in the timed region)
    if pred:
        line["predict"] = pred
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mra", choices=["mra", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=list(synth.SPECS))
    ap.add_argument("--n", type=int, default=None, help="override the config's n (same recipe)")
    ap.add_argument("--M", type=int, default=None, help="override the config's M (with --n: same leaf sizes)")
    ap.add_argument("--theta-lanes", type=int, default=None, help="plan option theta_lanes (NEXT-3): concurrent "
                    "evaluation contexts for a theta sweep (C4: no gain, its phases already fill the GPU; see DESIGN.md)")
    ap.add_argument("--stream-prior", type=int, default=0, help="plan option stream_prior (NEXT-4): 0 auto, "
                    "1 always, -1 never")
    ap.add_argument("--graph", type=int, default=0, help="plan option graph: log-L evaluations on device y replayed as "
                    "a CUDA graph (theta from device memory); measured no faster: C0 0.98 -> 1.24 ms, C1 3.15 -> 3.10, C2 equal")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle CPU work")
    ap.add_argument("--ref-budget", type=float, default=10.0, help="seconds of oracle work per reference step")
    ap.add_argument("--predict", type=int, default=0, help="also time mra_predict at this many random query "
                    "locations (1 GPU; after one posterior-state evaluation); adds a 'predict' key")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "mra":
        # `python bench.py --gpus N`: one process per GPU, launched here the way the driver launches it
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        if torch.cuda.device_count() < world:
            raise SystemExit(f"--gpus {world} needs {world} visible GPUs, found {torch.cuda.device_count()}")
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
