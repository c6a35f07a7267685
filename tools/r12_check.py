"""DESIGN.md R12: who carries the posterior-mean error on the conditioning-limited Matern case?
Compares the GPU path and the fp64 oracle against the extended-precision build of the same oracle loops
(oracle.run(..., extended=True)), per level of the tree. Usage: python tools/r12_check.py [wide]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402

CASES = [(2000, 7, 4, 16, 1, 0), (4000, 5, 2, 30, 1, 0), (2000, 7, 4, 16, 0, 0), (6000, 6, 4, 36, 1, 0)]


def levels(J, M, rh):
    out, f = [], 0
    for m in range(1, M):
        c = J ** (m - 1)
        out.append((m, f * rh, (f + c) * rh))
        f += c
    return out


def main():
    import paper_1905_00141_b200 as mra
    mra.load_library()
    wide = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    res = []
    for (n, M, J, r, cov, cl) in CASES:
        x, y, z = synth.uniform_small(n, seed=700 + n, clusters=cl)
        th = (cov, 1.1, 0.3, 0.07)
        d = oracle.run(x, y, z, M, J, r, th, posterior=True)
        e = oracle.run(x, y, z, M, J, r, th, posterior=True, extended=True)
        p = mra.mra_plan_create(x, y, M, J, r, wide=wide)
        g = mra.mra_loglik(p, z, th, posterior=True)
        mu_e = e["mu"].ravel()
        den = np.max(np.abs(mu_e))
        row = {"case": [n, M, J, r, cov], "max_abs_mu": float(den),
               "loglik_rel": {"oracle64": abs(d["loglik"] - e["loglik"]) / abs(e["loglik"]),
                              "gpu": abs(g["loglik"] - e["loglik"]) / abs(e["loglik"])},
               "mu_normwise": {"oracle64": float(np.max(np.abs(d["mu"].ravel() - mu_e)) / den),
                               "gpu": float(np.max(np.abs(g["mu"].ravel() - mu_e)) / den)},
               "smooth_normwise": {
                   "oracle64": float(np.nanmax(np.abs(d["smooth"] - e["smooth"])) / np.nanmax(np.abs(e["smooth"]))),
                   "gpu": float(np.nanmax(np.abs(g["smooth"] - e["smooth"])) / np.nanmax(np.abs(e["smooth"])))},
               "per_level_mu": []}
        for m, a, b in levels(J, M, p.r_hat):
            row["per_level_mu"].append({"level": m, "max_abs": float(np.max(np.abs(mu_e[a:b]))),
                                        "oracle64": float(np.max(np.abs(d["mu"].ravel()[a:b] - mu_e[a:b])) / den),
                                        "gpu": float(np.max(np.abs(g["mu"].ravel()[a:b] - mu_e[a:b])) / den)})
        res.append(row)
        print(json.dumps(row), flush=True)
        p.close()


if __name__ == "__main__":
    main()
