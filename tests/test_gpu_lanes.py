"""Theta-batched sweeps: a plan with theta_lanes = k keeps k
evaluation contexts and mra_loglik_batch* evaluates k parameter sets concurrently on k streams. Each
evaluation runs the same kernels on the same task lists as a one-lane plan, so the log-likelihoods are
bitwise equal to the sequential sweep, and within the north_star tolerance of the oracle."""
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


def _thetas(cov, k):
    rng = np.random.default_rng(7)
    return [(cov, float(s), float(r), float(t)) for s, r, t in
            zip(rng.uniform(0.5, 2.0, k), rng.uniform(0.05, 0.4, k), rng.uniform(0.01, 0.2, k))]


@pytest.mark.parametrize("lanes,ntheta", [(2, 5), (3, 7), (4, 4)])
def test_lanes_equal_sequential_and_oracle(mra, lanes, ntheta):
    import torch
    w = synth.make("C4", n=30000)
    th = _thetas(EXP, ntheta)
    seq = mra.mra_plan_create(w.x, w.y, 7, w.J, w.r, theta_lanes=1)
    par = mra.mra_plan_create(w.x, w.y, 7, w.J, w.r, theta_lanes=lanes)
    zd = torch.from_numpy(w.z).cuda()
    a = mra.mra_loglik_batch_dev(seq, zd, th)
    b = mra.mra_loglik_batch_dev(par, zd, th)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(mra.mra_loglik_batch(par, w.z, th), b)    # host-y entry
    for t, g in zip(th[:2], b[:2]):
        ref = oracle.run(w.x, w.y, w.z, 7, w.J, w.r, t)["loglik"]
        assert abs(g - ref) <= 1e-9 * abs(ref)
    # the single-evaluation entry points still work on a laned plan
    assert mra.mra_loglik_dev(par, zd, th[0])["loglik"] == a[0]


@pytest.mark.parametrize("wide", [0, -1])
def test_lanes_wide_and_bottom_paths(mra, wide):
    import torch
    x, y, z = synth.uniform_small(12000, seed=41, clusters=3)
    th = _thetas(MAT, 6)
    seq = mra.mra_plan_create(x, y, 5, 4, 25, wide=wide)
    par = mra.mra_plan_create(x, y, 5, 4, 25, wide=wide, theta_lanes=3)
    zd = torch.from_numpy(z).cuda()
    np.testing.assert_array_equal(mra.mra_loglik_batch_dev(seq, zd, th), mra.mra_loglik_batch_dev(par, zd, th))


def test_lanes_memory_profile_and_errors(mra):
    import torch
    x, y, z = synth.uniform_small(8000, seed=42)
    p1 = mra.mra_plan_create(x, y, 4, 4, 16, mem_budget_gb=0.5)
    p3 = mra.mra_plan_create(x, y, 4, 4, 16, mem_budget_gb=0.5, theta_lanes=3)
    assert mra.mra_plan_memory(p3)["device_bytes"] > mra.mra_plan_memory(p1)["device_bytes"]
    zd = torch.from_numpy(z).cuda()
    th = _thetas(EXP, 6)
    mra.mra_profile(p3, True)
    mra.mra_loglik_batch_dev(p3, zd, th)
    t = mra.mra_kernel_times(p3)
    mra.mra_profile(p3, False)
    n_prior = t["prior"][1]
    seq_launch = mra.mra_plan_create(x, y, 4, 4, 16)
    mra.mra_profile(seq_launch, True)
    mra.mra_loglik_dev(seq_launch, zd, th[0])
    assert n_prior == 6 * mra.mra_kernel_times(seq_launch)["prior"][1]   # every lane's launches counted
    assert mra.mra_last_launches(p3) == 6 * mra.mra_last_launches(seq_launch)
    bad = list(th)
    bad[4] = (EXP, 1.0, -0.1, 0.05)
    with pytest.raises(mra.MraError) as e:
        mra.mra_loglik_batch_dev(p3, zd, bad)
    assert e.value.status == 1
    np.testing.assert_array_equal(mra.mra_loglik_batch_dev(p3, zd, th[:3]), mra.mra_loglik_batch_dev(p1, zd, th[:3]))


def test_optimizer_on_laned_plan(mra):
    """mra_optimize evaluates its initial simplex and shrink points as one sweep on a laned plan:
    same evaluations, same decisions, bitwise the same optimum."""
    import torch
    x, y, z = synth.uniform_small(6000, seed=43)
    zd = torch.from_numpy(z).cuda()
    th0 = (EXP, 1.0, 0.1, 0.05)
    a = mra.mra_optimize(mra.mra_plan_create(x, y, 4, 4, 16), zd, th0, max_evals=40)
    b = mra.mra_optimize(mra.mra_plan_create(x, y, 4, 4, 16, theta_lanes=4), zd, th0, max_evals=40)
    assert tuple(a[0]) == tuple(b[0]) and a[1] == b[1] and a[2] == b[2]


def test_lanes_on_streaming_multichunk_plan(mra):
    """Lanes of a plan that streams its prior per chunk (NEXT-4) and runs many chunks: each lane owns its
    chunk-sized prior buffer; the sweep equals the resident one-lane plan bitwise."""
    import torch
    x, y, z = synth.uniform_small(10000, seed=44, clusters=2)
    th = _thetas(EXP, 5)
    ref = mra.mra_plan_create(x, y, 5, 4, 16, stream_prior=-1)
    par = mra.mra_plan_create(x, y, 5, 4, 16, stream_prior=1, mem_budget_gb=0.008, theta_lanes=2)
    info = mra.mra_plan_memory(par)
    assert info["streams_prior"] and info["chunk_regions"] < 4 ** (info["chunk_level"] - 1)
    zd = torch.from_numpy(z).cuda()
    np.testing.assert_array_equal(mra.mra_loglik_batch_dev(ref, zd, th), mra.mra_loglik_batch_dev(par, zd, th))


def test_numeric_failure_is_reported_and_plan_recovers(mra):
    """A parameter set whose leaf covariance is numerically singular (50 copies of one location and a
    nugget of 1e-30) makes a Cholesky pivot non-positive: MRA_E_NUMERIC naming the region, in single
    evaluations and inside a laned sweep; the plan evaluates the next parameter set correctly."""
    import torch
    x, y, z = synth.uniform_small(3000, seed=45)
    x[:50] = 0.3141
    y[:50] = 0.2718
    good = (EXP, 1.0, 0.1, 0.05)
    bad = (EXP, 1.0, 0.1, 1e-30)
    ref = mra.mra_loglik(mra.mra_plan_create(x, y, 4, 4, 16), z, good)["loglik"]
    zd = torch.from_numpy(z).cuda()
    for lanes in (1, 3):
        p = mra.mra_plan_create(x, y, 4, 4, 16, theta_lanes=lanes)
        with pytest.raises(mra.MraError) as e:
            mra.mra_loglik_dev(p, zd, bad)
        assert e.value.status == 4 and "Cholesky" in str(e.value)
        with pytest.raises(mra.MraError) as e:
            mra.mra_loglik_batch_dev(p, zd, [good, bad, good, good])
        assert e.value.status == 4
        assert mra.mra_loglik_dev(p, zd, good)["loglik"] == ref
        np.testing.assert_array_equal(mra.mra_loglik_batch_dev(p, zd, [good, good, good]), [ref, ref, ref])
