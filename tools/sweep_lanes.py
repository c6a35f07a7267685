"""Time a theta sweep (mra_loglik_batch_dev) on plans with 1..k theta lanes (NEXT-3 measurements)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_00141_b200 as mra  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C1")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--ntheta", type=int, default=16)
ap.add_argument("--lanes", default="1,2,4")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
w = synth.make(a.config, n=a.n, device="cuda")
rng = np.random.default_rng(3)
th0 = w.thetas[0]
thetas = [(th0[0], th0[1] * f1, th0[2] * f2, th0[3] * f3)
          for f1, f2, f3 in zip(rng.uniform(0.7, 1.4, a.ntheta), rng.uniform(0.7, 1.4, a.ntheta),
                                rng.uniform(0.7, 1.4, a.ntheta))]
zd = torch.from_numpy(w.z).cuda()
ref = None
for k in [int(v) for v in a.lanes.split(",")]:
    plan = mra.mra_plan_create(w.x, w.y, w.M, w.J, w.r, stream=torch.cuda.current_stream(), theta_lanes=k)
    ll = mra.mra_loglik_batch_dev(plan, zd, thetas)
    if ref is None:
        ref = ll
    same = bool(np.array_equal(ll, ref))
    ts = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        mra.mra_loglik_batch_dev(plan, zd, thetas)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"{a.config} n={w.n} thetas={a.ntheta} lanes={k}: {1e3 * min(ts):.2f} ms per sweep "
          f"({1e3 * min(ts) / a.ntheta:.3f} ms per theta), bitwise equal to 1 lane: {same}, "
          f"device {mra.mra_plan_memory(plan)['device_bytes'] / 1e9:.1f} GB")
    plan.close()
