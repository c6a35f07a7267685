"""mra_optimize (the paper's "optimization" mode) against scipy's Nelder-Mead on the
ORACLE's log-likelihood (oracle.run) for the same data: both maximise the same function, so the optima
must agree (log L to 1e-7 relative, parameters to 2e-3 relative), and the returned log L must be the
GPU evaluation at the returned theta."""
import numpy as np
import pytest
import scipy.optimize

import oracle
from oracle import dense

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mra():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1905_00141_b200 import build
    build.build()
    import paper_1905_00141_b200 as m
    m.load_library()
    return m


def test_optimize_matches_oracle_optimum(mra):
    import torch
    rng = np.random.default_rng(12)
    n = 1200
    x, y = rng.random(n), rng.random(n)
    C = 1.0 * np.exp(-dense.dist(x, y, x, y) / 0.1) + 0.05 * np.eye(n)
    z = np.linalg.cholesky(C) @ rng.standard_normal(n)
    M, J, r = 3, 4, 16
    lo, hi = (0.05, 0.005, 0.001), (20.0, 2.0, 2.0)
    p = mra.mra_plan_create(x, y, M, J, r)
    zd = torch.from_numpy(z).cuda()
    th, ll, ne = mra.mra_optimize(p, zd, (0, 0.5, 0.05, 0.2), lower=lo, upper=hi, max_evals=400, tol=1e-7)
    assert ne <= 400 and np.isfinite(ll)
    assert abs(mra.mra_loglik(p, z, th)["loglik"] - ll) <= 1e-12 * abs(ll)

    def negll(v):
        s2, rho, t2 = np.exp(v)
        return -oracle.run(x, y, z, M, J, r, (0, s2, rho, t2))["loglik"]

    res = scipy.optimize.minimize(negll, np.log([0.5, 0.05, 0.2]), method="Nelder-Mead",
                                  options=dict(xatol=1e-7, fatol=1e-10, maxiter=2000))
    ref = np.exp(res.x)
    assert abs(ll - (-res.fun)) <= 1e-7 * abs(res.fun)
    np.testing.assert_allclose(np.array(th[1:]), ref, rtol=2e-3)
    p.close()
