"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the pin (SURVEY.md §8(c) P1-P10 / DESIGN.md §4) and the passage it follows.
The oracle recursion (oracle/mra_oracle.c) and the dense definition (oracle/dense.py) are
independent implementations (separate partition code too); the dense definition is itself
pinned by P1 (library GP log-density), P4-P6 (closed-form properties of PAPER.md:84-92).
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.stats

import oracle
import synth
from oracle import dense

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_facts.json")))
EXP, MAT = 0, 1


# ------------------------------------------------------------------ plan facts (P9)
def test_r_hat_table():
    """r -> r_hat for the paper's nine settings (both implementations)."""
    for M, r, rh in GOLD["r_to_rhat"]["rows"]:
        x, y, _ = synth.uniform_small(50, seed=1)
        assert oracle.plan(x, y, 2, 2, r)["r_hat"] == rh
        assert dense.Tree(x, y, 2, 2, r).rh == rh


def test_knot_example_fig2():
    """PAPER.md:125 worked example: [0,1]^2, r=32, offset=0.1 -> 6 x 5 = 30 knots."""
    g = GOLD["knot_example"]
    t = dense.Tree(np.array([0.0, 1.0]), np.array([0.0, 1.0]), 1, 4, g["r"], g["offset"])
    assert (t.nx, t.ny, t.rh) == (g["nx"], g["ny"], g["r_hat"])
    np.testing.assert_allclose(t.bars(0.0, 1.0, t.nx), g["x_bars"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(t.bars(0.0, 1.0, t.ny), g["y_bars"], rtol=0, atol=1e-15)
    # the C oracle: root box of points {0,1}^2 is [0,1.01]^2, so scale the bars accordingly
    x = np.array([0.0, 1.0, 0.0, 1.0]); y = np.array([0.0, 0.0, 1.0, 1.0])
    p = oracle.plan(x, y, 2, 4, g["r"], offset=g["offset"])
    ext = 1.01
    np.testing.assert_allclose(np.unique(p["knots_x"][0]), np.array(g["x_bars"]) * ext, atol=1e-15)
    np.testing.assert_allclose(np.unique(p["knots_y"][0]), np.array(g["y_bars"]) * ext, atol=1e-15)


def test_region_counts():
    """J=2, M=10 -> 1023 / 512; M=14 -> 16,383 / 8,192."""
    x, y, _ = synth.uniform_small(64, seed=2)
    for J, M, tot, fin in GOLD["region_counts"]["rows"]:
        p = oracle.plan(x, y, M, J, 4)
        assert p["n_regions"] == tot
        assert p["n_regions"] - (J ** (M - 1) - 1) // (J - 1) == fin


def test_default_offset():
    assert abs(oracle.E_OVER_100 - GOLD["default_offset"]["value"]) <= 4e-18  # 1 ulp


def test_partition_geometry_and_membership():
    """children tile the parent (J=4 quadrants; J=2 halves of the longer axis),
    root = bbox with top/right pushed out 1%, half-open membership; C oracle == Python tree."""
    for J in (2, 4):
        x, y, _ = synth.uniform_small(2000, seed=3 + J, domain=(-3.0, 5.0, 10.0, 11.0))
        M = 5 if J == 4 else 7
        p = oracle.plan(x, y, M, J, 9)
        tr = dense.Tree(x, y, M, J, 9)
        b = p["boxes"]
        assert b[0, 0] == x.min() and b[0, 2] == y.min()
        assert b[0, 1] == x.max() + 0.01 * (x.max() - x.min())
        assert b[0, 3] == y.max() + 0.01 * (y.max() - y.min())
        for (m, t), bb in tr.boxes.items():
            rid = (J ** (m - 1) - 1) // (J - 1) + t
            assert tuple(b[rid]) == bb
            if m < M:
                kids = [tr.boxes[(m + 1, t * J + c)] for c in range(J)]
                area = sum((k[1] - k[0]) * (k[3] - k[2]) for k in kids)
                assert math.isclose(area, (bb[1] - bb[0]) * (bb[3] - bb[2]), rel_tol=1e-12)
                if J == 2:
                    longer_x = (bb[1] - bb[0]) >= (bb[3] - bb[2])
                    assert (kids[0][1] != bb[1]) == longer_x
        leaf = p["leaf"]
        np.testing.assert_array_equal(leaf, tr.leaf_of(x, y))
        lvlM = (J ** (M - 1) - 1) // (J - 1)
        for i in range(0, len(x), 97):
            bx = b[lvlM + leaf[i]]
            assert bx[0] <= x[i] < bx[1] and bx[2] <= y[i] < bx[3]


def test_half_open_shared_edges():
    """A point on an internal boundary belongs to the upper/right child only."""
    x = np.array([0.0, 1.0, 0.5, 0.5, 0.25]); y = np.array([0.0, 1.0, 0.5, 0.2, 0.5])
    p = oracle.plan(x, y, 2, 4, 4)
    mx = 0.5 * (0 + 1.01)
    # 0.5 < mx so (0.5,0.5) is SW; build a point exactly on the midline instead
    x2 = np.append(x, mx); y2 = np.append(y, mx)
    p = oracle.plan(x2, y2, 2, 4, 4)
    assert p["leaf"][-1] == 3                       # on both midlines -> NE
    tr = dense.Tree(x2, y2, 2, 4, 4)
    assert tr.region_at(mx, mx, 2) == 3


def test_knots_distinct_across_levels():
    """PAPER.md:135, Appendix A: with offset e/100 no two pre-finest knots
    coincide; with a rational offset the Appendix-A equation can be satisfied."""
    x, y, _ = synth.uniform_small(10, seed=4)
    for J, M, r in [(4, 5, 16), (2, 8, 9), (4, 4, 64), (2, 7, 30)]:
        p = oracle.plan(x, y, M, J, r)
        pts = set(zip(p["knots_x"].ravel().tolist(), p["knots_y"].ravel().tolist()))
        assert len(pts) == p["knots_x"].size
    # rational offset 0.25, r=9 (3 bars): the middle bar of a parent and the middle bar of ...
    # a J=4 child coincide with the parent's first/last bars: 0.25 of [0,1] == 0.5 of [0,0.5]
    x = np.array([0.0, 1.0 / 1.01]); y = np.array([0.0, 1.0 / 1.01])
    p = oracle.plan(x, y, 3, 4, 9, offset=0.25)
    pts = list(zip(p["knots_x"].ravel().tolist(), p["knots_y"].ravel().tolist()))
    assert len(set(pts)) < len(pts)


def test_elimination_of_obs_at_knots():
    """an observation located exactly at a pre-finest knot is eliminated."""
    x, y, z = synth.uniform_small(200, seed=5)
    p = oracle.plan(x, y, 3, 4, 9)
    kx, ky = p["knots_x"][2, 4], p["knots_y"][2, 4]        # a level-2 knot
    x2 = np.append(x, kx); y2 = np.append(y, ky); z2 = np.append(z, 1.0)
    p2 = oracle.plan(x2, y2, 3, 4, 9)
    assert p2["leaf"][-1] == -1 and (p2["leaf"][:-1] >= 0).all()
    o = oracle.run(x2, y2, z2, 3, 4, 9, (EXP, 1.0, 0.2, 0.1))
    o0 = oracle.run(x, y, z, 3, 4, 9, (EXP, 1.0, 0.2, 0.1))
    assert o["n_retained"] == 200
    assert abs(o["loglik"] - o0["loglik"]) < 1e-12 * abs(o0["loglik"])


# -------------------------------------------------------------- the recursion (P1, P2)
def test_P1_M1_is_exact_gp():
    """P1: with M=1 all observations are the (only) knots, so log L is the exact dense GP
    log-likelihood (scipy.stats.multivariate_normal) of C + tau2 I."""
    for cov in (EXP, MAT):
        x, y, z = synth.uniform_small(300, seed=6 + cov)
        th = (cov, 1.3, 0.15, 0.07)
        o = oracle.run(x, y, z, 1, 4, 16, th)
        C = dense.cov(dense.dist(x, y, x, y), cov, 1.3, 0.15) + 0.07 * np.eye(300)
        ref = scipy.stats.multivariate_normal(np.zeros(300), C).logpdf(z)
        assert abs(o["loglik"] - ref) <= 1e-12 * abs(ref)


CASES = [  # (n, M, J, r, cov, clusters)
    (300, 2, 4, 9, EXP, 0), (362, 3, 4, 9, EXP, 0), (300, 4, 2, 4, EXP, 0),
    (430, 3, 4, 16, EXP, 3), (250, 4, 2, 9, MAT, 2), (400, 3, 4, 36, MAT, 0),
    (260, 5, 2, 6, EXP, 0), (500, 2, 2, 30, EXP, 4),
]


@pytest.mark.parametrize("n,M,J,r,cov,cl", CASES)
def test_P2_recursion_equals_dense_definition(n, M, J, r, cov, cl):
    """P2: log L, log|Sigma_MRA + tau2 I| (= d_root) and y^T(...)^{-1}y (= u_root) of the
    recursion equal the dense Sigma_MRA of PAPER.md:62-92 (incl. empty leaves when clustered)."""
    x, y, z = synth.uniform_small(n, seed=n + 7 * M + J, clusters=cl)
    th = (cov, 1.0, 0.12, 0.05)
    o = oracle.run(x, y, z, M, J, r, th)
    ref = dense.loglik(x, y, z, M, J, r, cov, 1.0, 0.12, 0.05)
    ld, qf = dense.logdet_quad(x, y, z, M, J, r, cov, 1.0, 0.12, 0.05)
    assert abs(o["loglik"] - ref) <= 1e-12 * abs(ref)
    assert abs(o["d"] - ld) <= 1e-11 * max(1.0, abs(ld))
    assert abs(o["u"] - qf) <= 1e-11 * max(1.0, abs(qf))


def test_P2_empty_leaves_present():
    """The clustered cases above really contain empty leaves (PAPER.md:535 saw 30)."""
    x, y, z = synth.uniform_small(430, seed=430 + 21 + 4, clusters=3)
    p = oracle.plan(x, y, 3, 4, 16)
    assert len(np.unique(p["leaf"])) < 16


# ------------------------------------------------------- properties of Sigma_MRA (P3-P6)
def _sig_all(n=260, M=3, J=4, r=9, cov=EXP, seed=11):
    x, y, z = synth.uniform_small(n, seed=seed)
    return dense.sigma_mra(x, y, M, J, r, cov, 1.0, 0.2, return_all=True) + (x, y)


def test_P3_sigma_mra_spd():
    Sig, keep, nobs, ks, tree, x, y = _sig_all()
    S = Sig[:nobs, :nobs]
    assert np.abs(S - S.T).max() < 1e-14
    assert np.linalg.eigvalsh(S).min() > 0


def test_P4_same_leaf_pairs_reproduce_C():
    """Telescoping of PAPER.md:84-92: for two observations in the same finest region the sum
    of all levels equals C exactly; the diagonal equals sigma2."""
    Sig, keep, nobs, ks, tree, x, y = _sig_all()
    leaf = tree.leaf_of(x, y)[keep]
    C = dense.cov(dense.dist(x[keep], y[keep], x[keep], y[keep]), EXP, 1.0, 0.2)
    same = leaf[:, None] == leaf[None, :]
    assert np.abs((Sig[:nobs, :nobs] - C)[same]).max() < 1e-13
    assert np.abs(np.diag(Sig[:nobs, :nobs]) - 1.0).max() < 1e-13


def test_P5_knot_exactness():
    """north_star: Sigma_MRA reproduces C exactly on same-region knot pairs: for a knot q of a
    level-m region R and any point s in R, Sigma(q, s) = C(q, s) (C_{m+1}(q, .) = 0)."""
    Sig, keep, nobs, ks, tree, x, y = _sig_all(M=4, J=2, r=4)
    zx = np.concatenate([x[keep]] + [tree.knots(m, t)[0] for (m, t) in ks])
    zy = np.concatenate([y[keep]] + [tree.knots(m, t)[1] for (m, t) in ks])
    C = dense.cov(dense.dist(zx, zy, zx, zy), EXP, 1.0, 0.2)
    worst = 0.0
    for (m, t), qidx in ks.items():
        b = tree.boxes[(m, t)]
        inR = np.nonzero((zx >= b[0]) & (zx < b[1]) & (zy >= b[2]) & (zy < b[3]))[0]
        worst = max(worst, np.abs(Sig[np.ix_(qidx, inR)] - C[np.ix_(qidx, inR)]).max())
    assert worst < 1e-13


def test_P6_cross_region_coupling_is_level1_only():
    """Observations in different level-2 regions couple only through tau_1:
    Sigma(s1, s2) = C(s1, Q_1) C(Q_1, Q_1)^{-1} C(Q_1, s2)."""
    Sig, keep, nobs, ks, tree, x, y = _sig_all(M=3, J=4, r=9)
    xs, ys = x[keep], y[keep]
    reg2 = np.array([tree.region_at(a, b, 2) for a, b in zip(xs, ys)])
    qx, qy = tree.knots(1, 0)
    CsQ = dense.cov(dense.dist(xs, ys, qx, qy), EXP, 1.0, 0.2)
    CQQ = dense.cov(dense.dist(qx, qy, qx, qy), EXP, 1.0, 0.2)
    T1 = CsQ @ np.linalg.solve(CQQ, CsQ.T)
    diff = reg2[:, None] != reg2[None, :]
    assert np.abs((Sig[:nobs, :nobs] - T1)[diff]).max() < 1e-13


# ----------------------------------------------------------------- posterior state (P7)
@pytest.mark.parametrize("n,M,J,r,cov,cl", [CASES[1], CASES[2], CASES[4], CASES[3]])
def test_P7_posterior_means(n, M, J, r, cov, cl):
    """E[X(s)|y] at observations and knots from the recursion's mu equal the dense
    Sigma[., obs] (Sigma_MRA + tau2 I)^{-1} y."""
    x, y, z = synth.uniform_small(n, seed=n + 7 * M + J, clusters=cl)
    th = (cov, 1.0, 0.12, 0.05)
    o = oracle.run(x, y, z, M, J, r, th, posterior=True)
    sm, xq = dense.posterior(x, y, z, M, J, r, cov, 1.0, 0.12, 0.05)
    scale = np.nanmax(np.abs(sm))
    assert np.nanmax(np.abs(o["smooth"] - sm)) <= 1e-12 * scale
    for (m, t), v in xq.items():
        rid = (J ** (m - 1) - 1) // (J - 1) + t
        assert np.abs(o["xq"][rid] - v).max() <= 1e-11 * max(1.0, np.abs(v).max())


# -------------------------------------------------------------------- invariances (P8)
def test_P8_invariances():
    x, y, z = synth.uniform_small(350, seed=21)
    th = (EXP, 1.0, 0.1, 0.05)
    base = oracle.run(x, y, z, 3, 4, 16, th)["loglik"]
    perm = np.random.default_rng(0).permutation(350)
    assert abs(oracle.run(x[perm], y[perm], z[perm], 3, 4, 16, th)["loglik"] - base) <= 1e-12 * abs(base)
    # translation by a dyadic amount keeps every split and knot exact
    tr = oracle.run(x + 4.0, y - 2.0, z, 3, 4, 16, th)["loglik"]
    assert abs(tr - base) <= 1e-11 * abs(base)
    # joint scaling of coordinates and rho by a power of two
    sc = oracle.run(8.0 * x, 8.0 * y, z, 3, 4, 16, (EXP, 1.0, 0.8, 0.05))["loglik"]
    assert abs(sc - base) <= 1e-12 * abs(base)


def test_P10_region_terms_subtree_mode():
    """Subtree evaluation (used for sampled parity at full size) reproduces the per-region d, u
    of the full evaluation; empty leaves contribute d = u = 0."""
    x, y, z = synth.uniform_small(600, seed=31, clusters=3)
    th = (EXP, 1.0, 0.1, 0.05)
    full = oracle.run(x, y, z, 4, 4, 9, th, regions=True)
    for (lvl, t) in [(2, 1), (3, 5), (4, 17), (4, 0)]:
        rid = (4 ** (lvl - 1) - 1) // 3 + t
        sub = oracle.run(x, y, z, 4, 4, 9, th, target=(lvl, t))
        assert abs(sub["d"] - full["region_d"][rid]) <= 1e-12 * max(1, abs(sub["d"]))
        assert abs(sub["u"] - full["region_u"][rid]) <= 1e-12 * max(1, abs(sub["u"]))
    leaf = oracle.plan(x, y, 4, 4, 9)["leaf"]
    empty = sorted(set(range(64)) - set(leaf.tolist()))
    assert empty
    for t in empty[:3]:
        rid = 21 + t
        assert full["region_d"][rid] == 0.0 and full["region_u"][rid] == 0.0


def test_eq1_atilde_bound():
    """Eq. (1) PAPER.md:488 evaluated for the paper's setups (printed in SPEC / BASELINE)."""
    for J, M, r, gib in GOLD["eq1_atilde_gib"]["rows"]:
        v = J ** (M - 1) * M * (M - 1) * r * r * 2.0 ** -28
        assert abs(v - gib) < 0.005


def test_c0_inputs_shape():
    w = synth.make("C0")
    assert w.n == 4096 and (w.M, w.J, w.r) == (3, 4, 16)
    o = oracle.run(w.x, w.y, w.z, w.M, w.J, w.r, w.thetas[0])
    assert o["n_retained"] == 4096 and np.isfinite(o["loglik"])


# ------------------------------------------------------ prediction (NEXT-1)
def _queries(x, y, seed, k=24):
    """Random interior points + points exactly at observations + points at level-1 knots."""
    rng = np.random.default_rng(seed)
    qx = np.concatenate([rng.uniform(x.min(), x.max(), k), x[:6]])
    qy = np.concatenate([rng.uniform(y.min(), y.max(), k), y[:6]])
    return qx, qy


@pytest.mark.parametrize("n,M,J,r,cov,cl", [
    (300, 3, 4, 9, EXP, 0), (250, 4, 2, 9, MAT, 2), (362, 3, 4, 16, EXP, 3),
    (300, 2, 2, 4, MAT, 0), (280, 5, 2, 4, EXP, 4)])
def test_P11_prediction_recursion_equals_dense_definition(n, M, J, r, cov, cl):
    """Prediction (PAPER.md:228 'prediction' mode): the recursion's posterior
    mean / variance of X at query points equal kriging with the explicitly assembled Sigma_MRA
    (queries joining Z as finest-level points) -- means and variances, incl.
    queries at observations and in empty leaves (clustered inputs)."""
    x, y, z = synth.uniform_small(n, seed=31 + n, clusters=cl)
    qx, qy = _queries(x, y, seed=n)
    p = dense.Tree(x, y, M, J, r)
    kx, ky = p.knots(1, 0)
    qx = np.concatenate([qx, kx[:3]]); qy = np.concatenate([qy, ky[:3]])
    th = (cov, 1.3, 0.12, 0.06)
    m1, v1 = oracle.predict(x, y, z, qx, qy, M, J, r, th)
    m2, v2 = dense.predict(x, y, z, qx, qy, M, J, r, cov, 1.3, 0.12, 0.06)
    assert np.max(np.abs(m1 - m2)) <= 1e-11 * np.max(np.abs(m2))
    assert np.max(np.abs(v1 - v2)) <= 1e-11 * 1.3
    assert np.all(v1 > 0) and np.all(v1 <= 1.3 * (1 + 1e-12))


def test_P11_prediction_M1_is_kriging():
    """M = 1: textbook simple kriging with the full covariance (no approximation)."""
    x, y, z = synth.uniform_small(240, seed=8)
    qx, qy = _queries(x, y, seed=2)
    s2, rho, t2 = 0.9, 0.2, 0.04
    m1, v1 = oracle.predict(x, y, z, qx, qy, 1, 4, 9, (EXP, s2, rho, t2))
    C = s2 * np.exp(-dense.dist(x, y, x, y) / rho) + t2 * np.eye(len(x))
    Cq = s2 * np.exp(-dense.dist(qx, qy, x, y) / rho)
    mean = Cq @ np.linalg.solve(C, z)
    var = s2 - np.einsum("ij,ji->i", Cq, np.linalg.solve(C, Cq.T))
    np.testing.assert_allclose(m1, mean, rtol=0, atol=1e-11 * np.max(np.abs(mean)))
    np.testing.assert_allclose(v1, var, rtol=0, atol=1e-12)


def test_P11_prediction_at_observations_equals_smoothing():
    """A query at an observation location is X(s_i) itself: its predictive mean is the smoothing
    mean E[X(s_i)|y] of the posterior pass (pinned by P7)."""
    x, y, z = synth.uniform_small(400, seed=9, clusters=2)
    th = (EXP, 1.0, 0.1, 0.05)
    ref = oracle.run(x, y, z, 4, 4, 9, th, posterior=True)
    m, v = oracle.predict(x, y, z, x[:50], y[:50], 4, 4, 9, th)
    ok = ~np.isnan(ref["smooth"][:50])
    np.testing.assert_allclose(m[ok], ref["smooth"][:50][ok], rtol=0, atol=1e-12)
    assert np.all(v[ok] < th[3])   # posterior variance below the nugget where the point is observed


def test_P11_prediction_far_from_data_reverts_to_prior():
    """d >> rho from every observation (inside the domain): mean -> 0, variance -> sigma^2."""
    rng = np.random.default_rng(4)
    x = np.concatenate([rng.uniform(0, 0.1, 200), [1.0]])
    y = np.concatenate([rng.uniform(0, 0.1, 200), [1.0]])
    z = rng.standard_normal(201)
    m, v = oracle.predict(x, y, z, np.array([0.9, 0.6]), np.array([0.1, 0.5]), 3, 4, 9, (EXP, 2.0, 0.01, 0.1))
    assert np.all(np.abs(m) < 1e-12) and np.all(np.abs(v - 2.0) < 1e-12)


def test_P11_prediction_outside_domain_is_nan():
    x, y, z = synth.uniform_small(100, seed=3)
    m, v = oracle.predict(x, y, z, np.array([x.max() * 2 + 1, x.mean()]), np.array([y.mean(), y.mean()]), 2, 4,
                          4, (EXP, 1.0, 0.1, 0.05))
    assert np.isnan(m[0]) and np.isnan(v[0]) and np.isfinite(m[1]) and np.isfinite(v[1])


@pytest.mark.parametrize("n,M,J,r,cov,cl", [(300, 3, 4, 9, 0, 0), (300, 4, 2, 4, 1, 2), (430, 3, 4, 16, 1, 0)])
def test_extended_precision_build_pins(n, M, J, r, cov, cl):
    """The extended-precision build of the oracle (referee of DESIGN.md R12) is the same recursion: it equals
    the dense definition of Sigma_MRA (P2) and the fp64 oracle on well-conditioned inputs, log L / d / u to
    1e-12 and the smoothed values to 1e-10."""
    x, y, z = synth.uniform_small(n, seed=60 + n, clusters=cl)
    theta = (cov, 1.0, 0.2, 0.1)
    e = oracle.run(x, y, z, M, J, r, theta, posterior=True, extended=True)
    d = oracle.run(x, y, z, M, J, r, theta, posterior=True)
    for k in ("loglik", "d", "u"):
        assert abs(e[k] - d[k]) <= 1e-12 * abs(d[k]), k
    assert np.nanmax(np.abs(e["smooth"] - d["smooth"])) <= 1e-10 * np.nanmax(np.abs(d["smooth"]))
    dn = dense.loglik(x, y, z, M, J, r, *theta)
    assert abs(e["loglik"] - dn) <= 1e-11 * abs(dn)


@pytest.mark.parametrize("xs,ys,J,cov", [(2.0, 0.5, 4, 0), (0.3, 1.7, 2, 1)])
def test_axis_scaled_distance_pins(xs, ys, J, cov):
    """Reading R4's per-axis distance scaling (C2's "Euclidean distance on scaled coordinates"):
    the oracle with xscale / yscale != 1 equals the dense definition with the same scaled distance, and
    scaling an axis is the same as scaling that coordinate with the knots (the partition is affine-invariant
    for power-of-two factors)."""
    x, y, z = synth.uniform_small(350, seed=81, clusters=2)
    theta = (cov, 1.2, 0.25, 0.06)
    got = oracle.run(x, y, z, 3, J, 9, theta, xscale=xs, yscale=ys)["loglik"]
    ref = dense.loglik(x, y, z, 3, J, 9, *theta, xs=xs, ys=ys)
    assert abs(got - ref) <= 1e-12 * abs(ref)
    unscaled = oracle.run(x, y, z, 3, J, 9, theta)["loglik"]
    assert abs(got - unscaled) > 1e-6 * abs(unscaled)          # the scaling is not a no-op
    # x scale 2 with a J=4 tree == the coordinates x * 2 (exact in binary), knots scaling along
    if J == 4 and xs == 2.0 and ys == 0.5:
        alt = oracle.run(x * 2.0, y * 0.5, z, 3, J, 9, theta)["loglik"]
        assert abs(got - alt) <= 1e-12 * abs(alt)


def test_single_bar_midpoint_R7():
    """DESIGN R7 / R5 / R6: one bar sits at the box midpoint. Boxes written out by hand from R8 / R9
    (points {0,1}^2: root [0, 1.01]^2, J = 4 children SW, SE, NW, NE split at 0.505): r = 1 gives r_hat = 1 and
    one knot at each interior region's centre; r = 2 gives 2 x-bars (R6: lo + off ext, hi - off ext) and 1 y-bar
    (the midpoint), knots row-major by (y, x). The midpoint is also the mean of R6's bar set for any bar count
    (R6's bars are symmetric about it), which the last check confirms on the oracle's 6 x 5 example."""
    x = np.array([0.0, 1.0, 0.0, 1.0]); y = np.array([0.0, 0.0, 1.0, 1.0])
    e = 1.01
    h = e / 2
    boxes = [(0.0, e, 0.0, e), (0.0, h, 0.0, h), (h, e, 0.0, h), (0.0, h, h, e), (h, e, h, e)]   # xlo, xhi, ylo, yhi
    off = oracle.E_OVER_100
    p1 = oracle.plan(x, y, 3, 4, 1)
    assert p1["r_hat"] == 1
    for k, (x0, x1, y0, y1) in enumerate(boxes):
        assert abs(p1["knots_x"][k, 0] - 0.5 * (x0 + x1)) <= 1e-15
        assert abs(p1["knots_y"][k, 0] - 0.5 * (y0 + y1)) <= 1e-15
    p2 = oracle.plan(x, y, 3, 4, 2)
    assert p2["r_hat"] == 2
    for k, (x0, x1, y0, y1) in enumerate(boxes):
        ex = x1 - x0
        np.testing.assert_allclose(p2["knots_x"][k], [x0 + off * ex, x1 - off * ex], rtol=0, atol=1e-15)
        np.testing.assert_allclose(p2["knots_y"][k], [0.5 * (y0 + y1)] * 2, rtol=0, atol=1e-15)
    p30 = oracle.plan(x, y, 2, 4, 32)
    assert abs(np.mean(np.unique(p30["knots_x"][0])) - h) <= 1e-15
    assert abs(np.mean(np.unique(p30["knots_y"][0])) - h) <= 1e-15
