"""Run a few MRA evaluations of a config on cuda:0 (for ncu / compute-sanitizer captures)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1905_00141_b200 as mra  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--evals", type=int, default=1)
ap.add_argument("--M", type=int, default=None)
ap.add_argument("--lib", default=None)
ap.add_argument("--wide", type=int, default=0)
ap.add_argument("--budget", type=float, default=0.0)
ap.add_argument("--prof", action="store_true", help="per-class device times of the last evaluation")
ap.add_argument("--stream", type=int, default=0, help="stream_prior: 0 auto, 1 always, -1 never (NEXT-4)")
a = ap.parse_args()
if a.lib:
    mra.load_library(a.lib)
w = synth.make(a.config, n=a.n, device="cuda")
M = a.M or w.M
plan = mra.mra_plan_create(w.x, w.y, M, w.J, w.r, stream=torch.cuda.current_stream(), wide=a.wide,
                           mem_budget_gb=a.budget, stream_prior=a.stream)
torch.cuda.synchronize()
print(f"plan: n={w.n} M={M} retained={plan.n_retained} memory={mra.mra_plan_memory(plan)} "
      f"torch max allocated {torch.cuda.max_memory_allocated() / 1e9:.1f} GB")
zd = torch.from_numpy(w.z).cuda()
for i in range(a.evals):
    if a.prof and i == a.evals - 1:
        mra.mra_profile(plan, True)
    t = time.time()
    ll = mra.mra_loglik_dev(plan, zd, w.thetas[0])["loglik"]
    torch.cuda.synchronize()
    print(f"eval {i}: loglik={ll:.10f} {1e3 * (time.time() - t):.1f} ms launches={mra.mra_last_launches(plan)}")
if a.prof:
    print("kernel classes (ms, launches):", {k: (round(v[0], 1), v[1]) for k, v in mra.mra_kernel_times(plan).items() if v[1]})
import ctypes  # noqa: E402
cyc = (ctypes.c_uint64 * 32)()
mra._lib.mra_debug_phase_cycles(cyc, 1)
tot = sum(cyc[:6])
if tot:
    names = ["chain", "sigma", "chol", "fwd", "syrk", "merge"]
    print("bottom phases (CTA-cycles share):", ", ".join(f"{n} {100 * cyc[i] / tot:.1f}%" for i, n in enumerate(names)))
    print("  chol split: small-factor+inverse {:.1f}%, panel {:.1f}%, trailing {:.1f}%".format(
        *(100 * cyc[i] / tot for i in (6, 7, 8))))
    print(f"  chol_inv_small calls={cyc[11]} cycles/call={cyc[10] / max(1, cyc[11]):.0f} load_block cycles/call={cyc[9] / max(1, cyc[11]):.0f}; "
          f"bottom kernel CTA-cycles={cyc[12]:.3g} phase sum={tot:.3g}")
if cyc[17] or cyc[21]:
    per = lambda a, b: cyc[a] / max(1, cyc[b])
    print(f"mtile per task (CTA cycles): T00 {per(16, 17):.0f} (n={cyc[17]}); F: wait {per(19, 21):.0f} gemm1 {per(18, 21):.0f} "
          f"gemm2 {per(20, 21):.0f} (n={cyc[21]}); O: gemm1 {per(22, 25):.0f} wait {per(23, 25):.0f} gemm2 {per(24, 25):.0f} (n={cyc[25]})")
if cyc[29]:
    print(f"chain per task: {cyc[28] / cyc[29]:.0f} cycles; in cta_gemm calls {cyc[26] / cyc[29]:.0f}; "
          f"sum of K/rh per task {cyc[27] / cyc[29]:.1f} (ideal DMMA cycles at 2 CTA/SM: {cyc[27] / cyc[29] * 2 * 4096:.0f})")
if cyc[31]:
    print(f"mtile last-row (a = nr-1) O tasks: {cyc[30] / cyc[31]:.0f} cycles each (n={cyc[31]})")
