"""Write the full-size golden values of BASELINE.json configs C2, C3, C4 into tests/golden/.

Every stored value comes from `oracle/` (the CPU recursion, oracle/mra_oracle.c) run on the
inputs `synth` generates on the CPU (bitwise reproducible across CPU instruction sets and
thread counts: torch's CPU cos and numpy's PCG64 are used, nothing from the CUDA path). Each
entry is keyed by the SHA-256 of the input arrays (x, y, z), the SHA-256 of the oracle source
and the oracle's thread count, so a test can tell a stale golden from a parity failure.

  C2  log L, root d / u, every region's d_R / u_R, mu (all interior regions), E[X(s_i)|y] at a
      fixed sample of 131,072 observations (+ the full-array max |ref| for the normwise bound)
  C3  log L, root d / u, d_R / u_R of levels 1..5
  C4  per theta (indices given on the command line, default the corners 0 3 12 15 first, then
      the rest): log L, root d / u, d_R / u_R of levels 1..7

Usage:  python tools/make_golden.py C2 C4:0,3,12,15 C3 C4:1,2,4,5,6,7,8,9,10,11,13,14
Each target is written as soon as it finishes (tests/golden/full_<cfg>[_t<k>].json/.npz).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
SMOOTH_SAMPLE = 131072


def input_sha(w) -> str:
    h = hashlib.sha256()
    for a in (w.x, w.y, w.z):
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def oracle_sha() -> str:
    with open(os.path.join(ROOT, "oracle", "mra_oracle.c"), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def smooth_sample(n: int) -> np.ndarray:
    return np.sort(np.random.default_rng(12345).choice(n, size=min(n, SMOOTH_SAMPLE), replace=False))


def levels_upto(J: int, L: int) -> int:
    """number of regions in levels 1..L (level-major numbering)"""
    return (J ** L - 1) // (J - 1)


def run_one(name: str, ti: int, posterior: bool, keep_levels: int, w=None):
    w = w if w is not None else synth.make(name)
    theta = w.thetas[ti]
    t0 = time.time()
    ref = oracle.run(w.x, w.y, w.z, w.M, w.J, w.r, theta, regions=True, posterior=posterior)
    dt = time.time() - t0
    nkeep = levels_upto(w.J, min(keep_levels, w.M))
    meta = dict(config=name, theta_index=ti, theta=list(theta), n=w.n, M=w.M, J=w.J, r=w.r,
                r_hat=ref["r_hat"], n_retained=ref["n_retained"], loglik=ref["loglik"], d=ref["d"],
                u=ref["u"], input_sha256=input_sha(w), oracle_sha256=oracle_sha(),
                oracle_threads=oracle.threads(), oracle_seconds=round(dt, 1),
                region_levels=min(keep_levels, w.M),
                region_d=[float(v) for v in ref["region_d"][:nkeep]],
                region_u=[float(v) for v in ref["region_u"][:nkeep]],
                written_by="tools/make_golden.py (oracle/ only)")
    stem = f"full_{name}" + (f"_t{ti}" if len(w.thetas) > 1 else "")
    if posterior:
        idx = smooth_sample(w.n)
        sm = ref["smooth"]
        np.savez_compressed(os.path.join(GOLD, stem + "_post.npz"), mu=ref["mu"],
                            region_d=ref["region_d"], region_u=ref["region_u"],
                            smooth_idx=idx, smooth=sm[idx])
        meta["smooth_absmax"] = float(np.nanmax(np.abs(sm)))
        meta["mu_absmax"] = float(np.max(np.abs(ref["mu"])))
        meta["post_file"] = stem + "_post.npz"
    with open(os.path.join(GOLD, stem + ".json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(f"{stem}: log L {ref['loglik']!r} in {dt:.1f} s ({oracle.threads()} threads)", flush=True)
    return w


def main(argv):
    targets = argv or ["C2", "C4:0,3,12,15", "C3"]
    cache = {}
    for t in targets:
        name, _, sel = t.partition(":")
        if name not in cache:
            cache.clear()
            cache[name] = synth.make(name)
        w = cache[name]
        idx = [int(s) for s in sel.split(",")] if sel else [0]
        for ti in idx:
            if name == "C2":
                run_one(name, ti, posterior=True, keep_levels=5, w=w)
            elif name == "C3":
                run_one(name, ti, posterior=False, keep_levels=5, w=w)
            else:
                run_one(name, ti, posterior=False, keep_levels=7, w=w)


if __name__ == "__main__":
    main(sys.argv[1:])
