"""The leaf V chains and Sigma tiles as one dataflow kernel (k_wide_chsig, MRA_CHSIG=1) against the oracle, and
bitwise against the separate chain / Sigma kernels (same tasks, same arithmetic; only the schedule differs). Lag 1
makes nearly every Sigma task wait on its leaf's chain tasks; lag 3 and 40 exercise the ordinary staggering."""
import os
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

EXP, MAT = 0, 1
# (n, M, J, r, covariance, clusters): many-leaf sub-chunks, leaves of 1 to ~11 row tiles, empty leaves (clusters)
CASES = [
    (20000, 4, 4, 30, EXP, 3),
    (12800, 5, 4, 64, EXP, 3),
    (6000, 5, 2, 36, MAT, 2),
    (3000, 3, 4, 16, EXP, 1),
]


def _run(tmp_path, env_extra, tag):
    env = dict(os.environ)
    env.pop("MRA_CHSIG", None)
    env.update(env_extra)
    f = str(tmp_path / f"{tag}.npz")
    r = subprocess.run([sys.executable, os.path.join(HERE, "_chsig_worker.py"), f], env=env, cwd=HERE,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    return np.load(f)


@pytest.mark.gpu
def test_chsig_vs_oracle_and_separate(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import oracle
    import synth
    base = _run(tmp_path, {"MRA_CHSIG": "0"}, "sep")
    for lag in ("1", "3", "40"):
        fused = _run(tmp_path, {"MRA_CHSIG": "1", "MRA_CS_LAG": lag}, f"cs{lag}")
        for k in base.files:
            assert np.array_equal(base[k], fused[k], equal_nan=True), (lag, k)
    for ci, (n, M, J, r, cov, cl) in enumerate(CASES):
        x, y, z = synth.uniform_small(n, seed=300 + n + M, clusters=cl)
        ref = oracle.run(x, y, z, M, J, r, (cov, 1.0, 0.08, 0.05), posterior=True)
        ll = float(base[f"ll{ci}"][0])
        assert abs(ll - ref["loglik"]) <= 1e-9 * abs(ref["loglik"]), (ci, ll, ref["loglik"])
        sm = base[f"sm{ci}"]
        assert np.nanmax(np.abs(sm - ref["smooth"])) <= 1e-8 * np.nanmax(np.abs(ref["smooth"])), ci
