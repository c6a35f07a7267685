"""Worker of tests/test_gpu_chsig.py: runs the wide path's cases in a process whose MRA_CHSIG / MRA_CS_LAG (read once
by the library) select the fused chain + Sigma dataflow or the separate kernels, and saves log L and the posterior."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1905_00141_b200 as mra  # noqa: E402
import synth  # noqa: E402

from test_gpu_chsig import CASES  # noqa: E402

out = {}
for ci, (n, M, J, r, cov, cl) in enumerate(CASES):
    x, y, z = synth.uniform_small(n, seed=300 + n + M, clusters=cl)
    theta = (cov, 1.0, 0.08, 0.05)
    p = mra.mra_plan_create(x, y, M, J, r)
    got = mra.mra_loglik(p, z, theta, posterior=True, regions=True)
    out[f"ll{ci}"] = np.array([got["loglik"]])
    out[f"mu{ci}"] = got["mu"]
    out[f"sm{ci}"] = got["smooth"]
    out[f"rd{ci}"] = got["region_d"]
    p.close()
np.savez(sys.argv[1], **out)
