"""GPU mra_predict vs the CPU oracle's prediction (oracle.predict, pinned to the dense definition
by tests/test_oracle_pins.py P11), element by element through the C-ABI.

Tolerance: posterior means relative 1e-8 (north_star), normwise max|diff| / max|ref|; variances
absolute 1e-8 * sigma^2 (a variance is a difference of O(sigma^2) terms, so its error scales with
sigma^2, not with the variance itself)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
EXP, MAT = 0, 1


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


def _queries(x, y, seed, k):
    rng = np.random.default_rng(seed)
    qx = np.concatenate([rng.uniform(x.min(), x.max(), k), x[:17], [x.max() * 3 + 1.0]])
    qy = np.concatenate([rng.uniform(y.min(), y.max(), k), y[:17], [y.mean()]])
    return qx, qy


def _check(mra, x, y, z, M, J, r, theta, k=400, seed=0, wide=0):
    qx, qy = _queries(x, y, seed, k)
    p = mra.mra_plan_create(x, y, M, J, r, wide=wide)
    got = mra.mra_loglik(p, z, theta, posterior=True)
    gm, gv = mra.mra_predict(p, qx, qy)
    rm, rv = oracle.predict(x, y, z, qx, qy, M, J, r, theta)
    p.close()
    assert np.array_equal(np.isnan(gm), np.isnan(rm)) and np.isnan(gm[-1])
    ok = ~np.isnan(rm)
    assert np.max(np.abs(gm[ok] - rm[ok])) <= 1e-8 * np.max(np.abs(rm[ok]))
    assert np.max(np.abs(gv[ok] - rv[ok])) <= 1e-8 * theta[1]
    assert np.isfinite(got["loglik"])


CASES = [  # n, M, J, r, cov, clusters: ragged leaves, empty leaves, both J, both kernels, M = 1
    (3000, 3, 4, 16, EXP, 0),
    (4000, 5, 2, 30, MAT, 2),
    (2500, 4, 4, 36, EXP, 3),
    (1500, 1, 4, 16, EXP, 0),
    (12800, 5, 4, 64, EXP, 3),
    (2000, 2, 2, 64, MAT, 2),
]


@pytest.mark.parametrize("wide", [0, -1])
@pytest.mark.parametrize("n,M,J,r,cov,cl", CASES)
def test_predict_parity(mra, n, M, J, r, cov, cl, wide):
    x, y, z = synth.uniform_small(n, seed=500 + n + M, clusters=cl)
    _check(mra, x, y, z, M, J, r, (cov, 1.2, 0.09, 0.04), seed=n, wide=wide)


def test_predict_needs_posterior_state(mra):
    x, y, z = synth.uniform_small(1000, seed=3)
    p = mra.mra_plan_create(x, y, 3, 4, 16)
    mra.mra_loglik(p, z, (EXP, 1.0, 0.1, 0.05))
    with pytest.raises(mra.MraError):
        mra.mra_predict(p, x[:4], y[:4])
    mra.mra_loglik(p, z, (EXP, 1.0, 0.1, 0.05), posterior=True)
    m, v = mra.mra_predict(p, x[:4], y[:4])
    assert np.all(np.isfinite(m)) and np.all(v > 0)
    p.close()


def test_predict_C1_full_size(mra):
    """C1 at full size (131,072 observations, M = 6, r_hat = 36): 3,000 random queries + observations."""
    w = synth.make("C1")
    _check(mra, w.x, w.y, w.z, w.M, w.J, w.r, w.thetas[0], k=3000, seed=1)


def test_prediction_at_observations_equals_smoothing(mra):
    """Two independent GPU paths to the same quantity: mra_predict at the observed locations (k_predict:
    query basis + back substitution) and the smoothed values of the evaluation (k_smooth): E[X(s_i) | y]."""
    x, y, z = synth.uniform_small(4000, seed=48, clusters=2)
    theta = (0, 1.0, 0.1, 0.05)
    for wide in (0, -1):
        p = mra.mra_plan_create(x, y, 5, 4, 16, wide=wide)
        post = mra.mra_loglik(p, z, theta, posterior=True)
        mean, var = mra.mra_predict(p, x, y)
        ok = ~np.isnan(post["smooth"])
        assert ok.sum() == p.n_retained
        np.testing.assert_allclose(mean[ok], post["smooth"][ok], rtol=1e-9, atol=1e-11)
        assert np.all(var[ok] >= -1e-12) and np.all(var[ok] <= 1.0 + 1e-12)
