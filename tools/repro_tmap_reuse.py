"""Reproducer of the stale tensor-map fault (fixed by k_tmap_neutralize at plan destruction): a plan created and
destroyed before a laned plan runs a sweep with a failing theta. Prints the statuses of each call."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1905_00141_b200 as mra, synth
mra.load_library()
x, y, z = synth.uniform_small(3000, seed=45)
x[:50] = 0.3141
y[:50] = 0.2718
good = (0, 1.0, 0.1, 0.05)
bad = (0, 1.0, 0.1, 1e-30)
ref = mra.mra_loglik(mra.mra_plan_create(x, y, 4, 4, 16), z, good)["loglik"]
zd = torch.from_numpy(z).cuda()
for lanes in (1, 3):
    p = mra.mra_plan_create(x, y, 4, 4, 16, theta_lanes=lanes)
    for name, fn in (("single bad", lambda: mra.mra_loglik_dev(p, zd, bad)["loglik"]),
                     ("batch gbgg", lambda: mra.mra_loglik_batch_dev(p, zd, [good, bad, good, good])),
                     ("single good", lambda: mra.mra_loglik_dev(p, zd, good)["loglik"]),
                     ("batch ggg", lambda: mra.mra_loglik_batch_dev(p, zd, [good, good, good]))):
        try:
            print(lanes, name, fn(), ref, flush=True)
        except Exception as e:
            print(lanes, name, "ERR", e, flush=True)
