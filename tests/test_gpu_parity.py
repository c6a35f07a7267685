"""GPU (sm_100a) path vs the CPU oracle, element by element, through the C-ABI.

Tolerances (BASELINE.json north_star): log L relative 1e-9; posterior means relative 1e-8
(normwise: max|diff| / max|ref|, reading R12). Per-region d_R, u_R (basis-invariant
terms) are compared with 1e-8 relative to max(1, |ref|).
"""
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


def _cmp(got, ref, posterior=True, regions=True, tol_ll=1e-9, tol_post=1e-8):
    rel = abs(got["loglik"] - ref["loglik"]) / abs(ref["loglik"])
    assert rel <= tol_ll, (got["loglik"], ref["loglik"], rel)
    if regions:
        rd, ru = ref["region_d"], ref["region_u"]
        ok = ~np.isnan(rd)
        assert np.all(np.abs(got["region_d"][ok] - rd[ok]) <= 1e-8 * np.maximum(1, np.abs(rd[ok])))
        assert np.all(np.abs(got["region_u"][ok] - ru[ok]) <= 1e-8 * np.maximum(1, np.abs(ru[ok])))
    if posterior:
        mu_r, mu_g = ref["mu"], got["mu"]
        if mu_r.size:
            assert np.max(np.abs(mu_g - mu_r)) <= tol_post * np.max(np.abs(mu_r))
        sm_r, sm_g = ref["smooth"], got["smooth"]
        assert np.array_equal(np.isnan(sm_r), np.isnan(sm_g))
        assert np.nanmax(np.abs(sm_g - sm_r)) <= tol_post * np.nanmax(np.abs(sm_r))


CASES = [  # n, M, J, r, cov, clusters  -- ragged tiles, empty leaves, both J, both kernels
    (3000, 3, 4, 16, EXP, 0),
    (5000, 4, 4, 36, EXP, 3),
    (4000, 5, 2, 30, MAT, 0),
    (2500, 6, 2, 9, EXP, 4),
    (6000, 3, 4, 64, MAT, 0),
    (1200, 2, 4, 25, EXP, 0),
    (2000, 2, 2, 64, EXP, 2),
    (9000, 4, 4, 30, EXP, 5),
    (12800, 5, 4, 64, EXP, 3),   # leaves 0..~600 around ncol = 257: both G = X[V|y] and blocked-solve leaves
    (4000, 6, 2, 36, MAT, 2),    # n_leaf <= ncol = 181 mostly: explicit-inverse path, 1-4 row blocks
]


@pytest.mark.parametrize("wide", [0, -1])
@pytest.mark.parametrize("n,M,J,r,cov,cl", CASES)
def test_parity_small(mra, n, M, J, r, cov, cl, wide):
    """Both schedules: the grid-wide task path (default) and one CTA per level-(M-1) region."""
    x, y, z = synth.uniform_small(n, seed=100 + n + M, clusters=cl)
    theta = (cov, 1.0, 0.08, 0.05)
    p = mra.mra_plan_create(x, y, M, J, r, wide=wide)
    got = mra.mra_loglik(p, z, theta, posterior=True, regions=True)
    ref = oracle.run(x, y, z, M, J, r, theta, regions=True, posterior=True)
    _cmp(got, ref)
    p.close()


def test_M1_exact_gp_large_leaf(mra):
    """M = 1: one leaf holding every observation; 1100 rows -> 18 Cholesky panels, ragged tail."""
    x, y, z = synth.uniform_small(1100, seed=5)
    theta = (EXP, 1.3, 0.2, 0.03)
    p = mra.mra_plan_create(x, y, 1, 4, 16)
    got = mra.mra_loglik(p, z, theta, posterior=True, regions=True)
    ref = oracle.run(x, y, z, 1, 4, 16, theta, regions=True, posterior=True)
    _cmp(got, ref)


def test_big_leaves_multi_panel(mra):
    """M = 2, J = 2: two leaves of ~700 observations (multi-panel Cholesky + forward substitution)."""
    x, y, z = synth.uniform_small(1400, seed=6)
    theta = (MAT, 2.0, 0.3, 0.1)
    p = mra.mra_plan_create(x, y, 2, 2, 49)
    got = mra.mra_loglik(p, z, theta, posterior=True, regions=True)
    ref = oracle.run(x, y, z, 2, 2, 49, theta, regions=True, posterior=True)
    _cmp(got, ref)


@pytest.mark.parametrize("wide", [0, -1])
def test_C0_full(mra, wide):
    w = synth.make("C0")
    p = mra.mra_plan_create(w.x, w.y, w.M, w.J, w.r, wide=wide)
    got = mra.mra_loglik(p, w.z, w.thetas[0], posterior=True, regions=True)
    ref = oracle.run(w.x, w.y, w.z, w.M, w.J, w.r, w.thetas[0], regions=True, posterior=True)
    _cmp(got, ref)


@pytest.mark.parametrize("wide", [0, -1])
def test_C1_full(mra, wide):
    w = synth.make("C1")
    p = mra.mra_plan_create(w.x, w.y, w.M, w.J, w.r, wide=wide)
    got = mra.mra_loglik(p, w.z, w.thetas[0], posterior=True, regions=True)
    ref = oracle.run(w.x, w.y, w.z, w.M, w.J, w.r, w.thetas[0], regions=True, posterior=True)
    _cmp(got, ref)


def test_device_and_host_entry_agree(mra):
    import torch
    x, y, z = synth.uniform_small(4000, seed=8)
    theta = (EXP, 1.0, 0.1, 0.05)
    p = mra.mra_plan_create(x, y, 4, 4, 16, stream=torch.cuda.current_stream())
    a = mra.mra_loglik(p, z, theta)["loglik"]
    zd = torch.from_numpy(z).cuda()
    b = mra.mra_loglik_dev(p, zd, theta)["loglik"]
    assert a == b                                      # same kernels, same order: bitwise
    c = mra.mra_loglik_dev(p, zd, theta)["loglik"]
    assert b == c                                      # deterministic run to run
    assert mra.mra_last_launches(p) > 0


def test_chunked_schedule_equals_single_chunk(mra):
    """A tiny memory budget forces a deeper chunk level and 1-region chunks."""
    x, y, z = synth.uniform_small(8000, seed=9, clusters=2)
    theta = (EXP, 1.0, 0.1, 0.05)
    p1 = mra.mra_plan_create(x, y, 5, 4, 16, wide=-1)
    p2 = mra.mra_plan_create(x, y, 5, 4, 16, mem_budget_gb=0.003, wide=-1)
    a = mra.mra_loglik(p1, z, theta, regions=True)
    b = mra.mra_loglik(p2, z, theta, regions=True)
    assert abs(a["loglik"] - b["loglik"]) <= 1e-12 * abs(a["loglik"])
    np.testing.assert_allclose(a["region_d"], b["region_d"], rtol=1e-12, atol=1e-12)


def test_sharded_algebra_on_one_gpu(mra):
    """Subtree sharding emulated on one GPU: each rank's shard pass runs to completion
    independently (no rank waits on another), the exchange buffers are summed (what ncclReduce does),
    rank 0 finishes. Must equal the single-GPU log L to 1e-12."""
    import torch
    x, y, z = synth.uniform_small(12000, seed=10, clusters=3)
    theta = (EXP, 1.0, 0.1, 0.05)
    single = mra.mra_loglik(mra.mra_plan_create(x, y, 5, 4, 16), z, theta)["loglik"]
    zd = torch.from_numpy(z).cuda()
    for world in (2, 3, 4):
        plans = [mra.mra_plan_create(x, y, 5, 4, 16, rank=r, world=world) for r in range(world)]
        size = mra.mra_shard_size(plans[0])
        total = torch.zeros(size, dtype=torch.float64, device="cuda")
        for pl in plans:
            buf = torch.zeros(size, dtype=torch.float64, device="cuda")
            mra.mra_loglik_shard(pl, zd, theta, buf)
            total += buf
        ll = mra.mra_loglik_finish(plans[0], theta, total)
        assert abs(ll - single) <= 1e-12 * abs(single), (world, ll, single)


@pytest.mark.parametrize("wide", [0, -1])
def test_sharded_posterior_on_one_gpu(mra, wide):
    """S6 on a sharded plan, ranks emulated in sequence on one GPU: shard passes keep
    their posterior state, rank 0 finishes and exports the above-shard means, every rank completes its
    own subtrees' means and smoothed values. The union over ranks equals the single-GPU posterior."""
    import torch
    x, y, z = synth.uniform_small(9000, seed=21, clusters=3)
    theta = (EXP, 1.0, 0.1, 0.05)
    M, J, r = 5, 4, 16
    p1 = mra.mra_plan_create(x, y, M, J, r, wide=wide)
    ref = mra.mra_loglik(p1, z, theta, posterior=True)
    p1.close()
    zd = torch.from_numpy(z).cuda()
    for world in (2, 3):
        plans = [mra.mra_plan_create(x, y, M, J, r, rank=k, world=world, wide=wide) for k in range(world)]
        size = mra.mra_shard_size(plans[0])
        total = torch.zeros(size, dtype=torch.float64, device="cuda")
        for pl in plans:
            buf = torch.zeros(size, dtype=torch.float64, device="cuda")
            mra.mra_loglik_shard_post(pl, zd, theta, buf)
            total += buf
        mutop = torch.empty(max(1, mra.mra_mutop_size(plans[0])), dtype=torch.float64, device="cuda")
        ll = mra.mra_loglik_finish_post(plans[0], theta, total, mutop)
        assert abs(ll - ref["loglik"]) <= 1e-12 * abs(ref["loglik"])
        nmu = plans[0].n_interior * plans[0].r_hat
        mu = np.full(nmu, np.nan)
        sm = np.full(len(x), np.nan)
        for pl in plans:
            dmu = torch.empty(nmu, dtype=torch.float64, device="cuda")
            dsm = torch.empty(len(x), dtype=torch.float64, device="cuda")
            mra.mra_posterior_shard(pl, mutop, dmu, dsm)
            m_, s_ = dmu.cpu().numpy(), dsm.cpu().numpy()
            mu = np.where(np.isnan(mu), m_, mu)
            sm = np.where(np.isnan(sm), s_, sm)
        ref_mu = ref["mu"].ravel()
        assert not np.any(np.isnan(mu))
        assert np.max(np.abs(mu - ref_mu)) <= 1e-10 * np.max(np.abs(ref_mu))
        assert np.array_equal(np.isnan(sm), np.isnan(ref["smooth"]))
        assert np.nanmax(np.abs(sm - ref["smooth"])) <= 1e-10 * np.nanmax(np.abs(ref["smooth"]))
        for pl in plans:
            pl.close()


def test_batch_thetas(mra):
    import torch
    w = synth.make("C4", n=30000)
    p = mra.mra_plan_create(w.x, w.y, 7, w.J, w.r)
    zd = torch.from_numpy(w.z).cuda()
    th = w.thetas[::5]
    got = mra.mra_loglik_batch_dev(p, zd, th)
    for t, g in zip(th, got):
        ref = oracle.run(w.x, w.y, w.z, 7, w.J, w.r, t)["loglik"]
        assert abs(g - ref) <= 1e-9 * abs(ref)
    np.testing.assert_array_equal(mra.mra_loglik_batch(p, w.z, th), got)   # host-y entry: same kernels


def test_bad_theta_is_arg_error(mra):
    x, y, z = synth.uniform_small(500, seed=11)
    p = mra.mra_plan_create(x, y, 3, 4, 16)
    for th in [(0, -1.0, 0.1, 0.1), (0, 1.0, 0.0, 0.1), (0, 1.0, 0.1, float("nan")), (7, 1.0, 0.1, 0.1)]:
        with pytest.raises(mra.MraError) as e:
            mra.mra_loglik(p, z, th)
        assert e.value.status == 1
    zb = z.copy(); zb[0] = np.inf
    with pytest.raises(mra.MraError):
        mra.mra_loglik(p, zb, (0, 1.0, 0.1, 0.1))


@pytest.mark.parametrize("n,M,J,r,cov,cl", [(6000, 3, 2, 30, EXP, 0), (9000, 4, 4, 16, MAT, 3), (3000, 2, 2, 64, EXP, 1),
                                            (12000, 5, 2, 25, EXP, 4)])
def test_wide_path_parity(mra, n, M, J, r, cov, cl):
    """Big-leaf path (all CTAs cooperate per leaf; forced on for moderate leaves so the oracle stays fast):
    multi-block left-looking Cholesky, ragged tails, empty leaves."""
    x, y, z = synth.uniform_small(n, seed=200 + n + M, clusters=cl)
    theta = (cov, 1.0, 0.08, 0.05)
    p = mra.mra_plan_create(x, y, M, J, r, wide=1)
    got = mra.mra_loglik(p, z, theta, posterior=False, regions=True)
    ref = oracle.run(x, y, z, M, J, r, theta, regions=True)
    _cmp(got, ref, posterior=False)
    # a tiny Sigma budget forces several sub-chunks
    p2 = mra.mra_plan_create(x, y, M, J, r, wide=1, mem_budget_gb=0.02)
    got2 = mra.mra_loglik(p2, z, theta)
    assert abs(got2["loglik"] - got["loglik"]) <= 1e-12 * abs(got["loglik"])


def test_wide_path_posterior(mra):
    """Posterior state (mu, smoothing) on a plan that takes the wide path."""
    x, y, z = synth.uniform_small(5000, seed=301, clusters=2)
    theta = (EXP, 1.0, 0.1, 0.05)
    p = mra.mra_plan_create(x, y, 3, 2, 30, wide=1)
    got = mra.mra_loglik(p, z, theta, posterior=True, regions=True)
    ref = oracle.run(x, y, z, 3, 2, 30, theta, regions=True, posterior=True)
    _cmp(got, ref)


@pytest.mark.parametrize("n,M,J,r,cl", [(5000, 4, 4, 16, 3), (4000, 6, 2, 9, 2), (3000, 1, 4, 16, 0),
                                        (20000, 7, 4, 36, 4)])
def test_device_plan_build_matches_host(mra, n, M, J, r, cl):
    """S0 on the device (NEXT-2): leaf keys, elimination and the stable sort give the host build's plan
    bit for bit (perm, CSR offsets, knots), hence the identical log L. Observations placed exactly on
    pre-finest knots exercise the elimination path."""
    x, y, z = synth.uniform_small(n, seed=900 + n, clusters=cl)
    ph = mra.mra_plan_create(x, y, M, J, r, host_plan=1)
    lh = mra.mra_plan_layout(ph)
    if M > 1:   # put 7 observations on level-1 / level-2 knots
        x = x.copy(); y = y.copy()
        k = min(7, lh["knots_x"].size)
        x[:k] = lh["knots_x"].ravel()[:k]
        y[:k] = lh["knots_y"].ravel()[:k]
        ph.close()
        ph = mra.mra_plan_create(x, y, M, J, r, host_plan=1)
        lh = mra.mra_plan_layout(ph)
    pd = mra.mra_plan_create(x, y, M, J, r)
    ld = mra.mra_plan_layout(pd)
    assert pd.n_retained == ph.n_retained and (M == 1 or pd.n_retained < n)
    for key in ("perm", "leaf_off", "knots_x", "knots_y"):
        assert np.array_equal(ld[key], lh[key]), key
    th = (EXP, 1.0, 0.1, 0.05)
    assert mra.mra_loglik(pd, z, th)["loglik"] == mra.mra_loglik(ph, z, th)["loglik"]
    pd.close(); ph.close()


@pytest.mark.parametrize("n,M,J,r,cov,cl,dom", [
    (800, 3, 4, 1, EXP, 0, (0.0, 1.0, 0.0, 1.0)),        # r_hat = 1: one knot per region (its midpoint, R7)
    (900, 4, 2, 2, MAT, 0, (0.0, 3.0, 0.0, 0.5)),        # r_hat = 2 (1 x 2 bars), wide flat domain: J=2 splits x
    (700, 3, 4, 3, EXP, 2, (-5.0, 5.0, 10.0, 11.0)),     # r_hat = 3, translated anisotropic domain, empty leaves
    (40, 2, 4, 4, EXP, 0, (0.0, 1.0, 0.0, 1.0)),         # ~10 observations per leaf
    (5, 2, 2, 4, MAT, 0, (0.0, 1.0, 0.0, 1.0)),          # 5 observations, most leaves empty or single
    (4000, 12, 2, 9, EXP, 3, (0.0, 1.0, 0.0, 1.0)),      # deep tree: 11 ancestor levels, 2,048 mostly empty leaves
    (2000, 7, 4, 16, EXP, 0, (0.0, 1.0, 0.0, 1.0)),      # 4,096 leaves for 2,000 observations
])
def test_edge_cases(mra, n, M, J, r, cov, cl, dom):
    """Degenerate knot counts (r_hat 1..3), extreme aspect ratios, tiny leaves, nearly-empty trees:
    log L, per-region terms and posterior state against the oracle."""
    x, y, z = synth.uniform_small(n, seed=700 + n, clusters=cl, domain=dom)
    theta = (cov, 1.1, 0.3, 0.07)
    for wide in (0, -1):
        p = mra.mra_plan_create(x, y, M, J, r, wide=wide)
        got = mra.mra_loglik(p, z, theta, posterior=True, regions=True)
        ref = oracle.run(x, y, z, M, J, r, theta, regions=True, posterior=True)
        _cmp(got, ref)
        p.close()


def test_nonfinite_inputs_are_arg_errors(mra):
    x, y, z = synth.uniform_small(300, seed=1)
    x2 = x.copy(); x2[5] = np.nan
    with pytest.raises(mra.MraError) as e:
        mra.mra_plan_create(x2, y, 3, 4, 9)
    assert e.value.status == 1
    with pytest.raises(mra.MraError) as e:
        mra.mra_plan_create(x2, y, 3, 4, 9, host_plan=1)
    assert e.value.status == 1
    p = mra.mra_plan_create(x, y, 3, 4, 9)
    z2 = z.copy(); z2[3] = np.inf
    with pytest.raises(mra.MraError) as e:
        mra.mra_loglik(p, z2, (EXP, 1.0, 0.1, 0.05))
    assert e.value.status == 1
    p.close()


def test_input_order_does_not_change_the_result(mra):
    """The plan sorts observations by leaf (stable on the input index): permuting the input permutes
    the smoothed values and leaves log L unchanged up to the within-leaf summation order."""
    x, y, z = synth.uniform_small(6000, seed=46, clusters=2)
    theta = (EXP, 1.0, 0.1, 0.05)
    a = mra.mra_loglik(mra.mra_plan_create(x, y, 5, 4, 16), z, theta, posterior=True)
    perm = np.random.default_rng(0).permutation(len(x))
    b = mra.mra_loglik(mra.mra_plan_create(x[perm], y[perm], 5, 4, 16), z[perm], theta, posterior=True)
    assert abs(a["loglik"] - b["loglik"]) <= 1e-12 * abs(a["loglik"])
    np.testing.assert_allclose(b["smooth"], a["smooth"][perm], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(b["mu"], a["mu"], rtol=1e-9, atol=1e-12)


def test_closed_form_invariances(mra):
    """Closed forms the MRA likelihood obeys exactly: scaling sigma2 and tau2 by c scales
    Sigma_MRA + tau2 I by c, so d' = d + N log c and u' = u / c; scaling the coordinates and rho by s
    leaves every covariance, the partition and the knots (relative to the bounding box) unchanged."""
    x, y, z = synth.uniform_small(5000, seed=47, clusters=2)
    p = mra.mra_plan_create(x, y, 5, 4, 16)
    a = mra.mra_loglik(p, z, (EXP, 1.3, 0.12, 0.04), posterior=True)
    c = 3.7
    b = mra.mra_loglik(p, z, (EXP, 1.3 * c, 0.12, 0.04 * c), posterior=True)
    N = p.n_retained
    assert abs(b["d"] - (a["d"] + N * np.log(c))) <= 1e-10 * abs(b["d"])
    assert abs(b["u"] - a["u"] / c) <= 1e-10 * abs(b["u"])
    np.testing.assert_allclose(b["smooth"], a["smooth"], rtol=1e-9, atol=1e-12)   # E[X|y] is scale-free
    s = 8.0   # a power of two: the scaled coordinates and knots are exact
    q = mra.mra_plan_create(x * s, y * s, 5, 4, 16)
    for cov in (EXP, MAT):
        la = mra.mra_loglik(p, z, (cov, 1.3, 0.12, 0.04))["loglik"]
        lb = mra.mra_loglik(q, z, (cov, 1.3, 0.12 * s, 0.04))["loglik"]
        assert abs(la - lb) <= 1e-12 * abs(la)


R12_CASES = [(2000, 7, 4, 16), (6000, 6, 4, 36), (4000, 5, 2, 30)]


@pytest.mark.parametrize("n,M,J,r", R12_CASES)
def test_conditioning_limited_posterior_means_R12(mra, n, M, J, r):
    """DESIGN.md R12: Matern-3/2 with rho = 0.3 down to small deep regions makes the paper-parametrization
    means mu_R = E[eta_R | y] ill-conditioned (|mu| up to ~300 from nearly collinear knot covariances). The
    referee is the extended-precision build of the oracle's own loops (oracle.run(extended=True)): against
    it the fp64 ORACLE misses the 1e-8 bound itself (7e-8 on the r = 36 case), so the GPU is held to the
    oracle's own fp64 accuracy -- within 4x of the fp64 oracle's error or 1e-8, whichever is larger --
    while log L (1e-9) and the smoothed values E[X(s_i)|y] (1e-8) keep the north_star bars."""
    x, y, z = synth.uniform_small(n, seed=700 + n)
    theta = (MAT, 1.1, 0.3, 0.07)
    ref = oracle.run(x, y, z, M, J, r, theta, posterior=True, extended=True)
    o64 = oracle.run(x, y, z, M, J, r, theta, posterior=True)
    den = np.max(np.abs(ref["mu"]))
    err64 = np.max(np.abs(o64["mu"] - ref["mu"])) / den
    for wide in (0, -1):
        p = mra.mra_plan_create(x, y, M, J, r, wide=wide)
        got = mra.mra_loglik(p, z, theta, posterior=True)
        assert abs(got["loglik"] - ref["loglik"]) <= 1e-9 * abs(ref["loglik"])
        assert np.nanmax(np.abs(got["smooth"] - ref["smooth"])) <= 1e-8 * np.nanmax(np.abs(ref["smooth"]))
        err = np.max(np.abs(got["mu"] - ref["mu"])) / den
        assert err <= max(1e-8, 4.0 * err64), (err, err64)
        p.close()


@pytest.mark.parametrize("xs,ys,J,cov", [(2.0, 0.5, 4, EXP), (0.3, 1.7, 2, MAT)])
def test_axis_scaled_distance(mra, xs, ys, J, cov):
    """opts.xscale / yscale (reading R4) on the GPU against the oracle with the same scaling (pinned to the
    dense definition in tests/test_oracle_pins.py)."""
    x, y, z = synth.uniform_small(6000, seed=83, clusters=2)
    theta = (cov, 1.2, 0.25, 0.06)
    for wide in (0, -1):
        p = mra.mra_plan_create(x, y, 4, J, 16, xscale=xs, yscale=ys, wide=wide)
        got = mra.mra_loglik(p, z, theta, posterior=True, regions=True)
        ref = oracle.run(x, y, z, 4, J, 16, theta, xscale=xs, yscale=ys, regions=True, posterior=True)
        _cmp(got, ref)
        p.close()


def test_graph_replay_equals_direct_launches(mra):
    """opts.graph: the evaluation captured once as a CUDA graph and replayed with theta read from device memory gives
    bitwise the direct launches' log L for several thetas of a family, re-captures for another family / y buffer,
    and posterior requests fall back to direct launches."""
    import torch
    x, y, z = synth.uniform_small(6000, seed=91, clusters=2)
    zd = torch.from_numpy(z).cuda()
    zd2 = zd.clone()
    pg = mra.mra_plan_create(x, y, 5, 4, 16, graph=True, stream=torch.cuda.current_stream())
    pd = mra.mra_plan_create(x, y, 5, 4, 16, stream=torch.cuda.current_stream())
    for th in [(EXP, 1.0, 0.1, 0.05), (EXP, 1.7, 0.05, 0.2), (MAT, 1.2, 0.2, 0.03), (EXP, 0.8, 0.3, 0.01)]:
        for y_dev in (zd, zd2):
            a = mra.mra_loglik_dev(pg, y_dev, th, regions=True)
            b = mra.mra_loglik_dev(pd, y_dev, th, regions=True)
            assert a["loglik"] == b["loglik"], th
            assert np.array_equal(a["region_d"], b["region_d"]) and np.array_equal(a["region_u"], b["region_u"])
            assert mra.mra_last_launches(pg) == mra.mra_last_launches(pd)
    ref = oracle.run(x, y, z, 5, 4, 16, (EXP, 0.8, 0.3, 0.01))["loglik"]
    assert abs(a["loglik"] - ref) <= 1e-9 * abs(ref)
    post = mra.mra_loglik_dev(pg, zd, (EXP, 1.0, 0.1, 0.05), posterior=True)
    postd = mra.mra_loglik_dev(pd, zd, (EXP, 1.0, 0.1, 0.05), posterior=True)
    assert torch.equal(post["smooth"], postd["smooth"])
    with pytest.raises(mra.MraError) as e:      # a failing Cholesky inside a replay is still reported
        mra.mra_loglik_dev(pg, zd, (EXP, 1.0, 0.1, -1.0))
    assert e.value.status == 1
