"""Dense DEFINITION of the MRA covariance -- TEST INFRASTRUCTURE ONLY.

Assembles Sigma_MRA explicitly for tiny inputs, exactly as PAPER.md:62-92 (§1.1)
defines it, and evaluates the Gaussian log-likelihood with a library routine:

  Z = retained observations  ∪  all knots of levels 1..M-1,   C^(1) = C(Z, Z)
  for m = 1..M-1:
      T^(m)[a,b] = 1[a,b in the same level-m region R] C^(m)(a,Q_R) C^(m)(Q_R,Q_R)^{-1} C^(m)(Q_R,b)
      Sigma     += T^(m)                               (tau_m, the level-m predictive process)
      C^(m+1)    = 1[same level-(m+1) region] (C^(m) - T^(m))   (delta_{m+1})
  Sigma += C^(M)                                        (tau_M: level-M knots = the observations,
                                                         PAPER.md:60, so tau_M = delta_M at them)
  Sigma_MRA = Sigma[obs, obs]

The partition and knots are re-implemented here in plain Python from PAPER.md:99-135
(independently of oracle/mra_oracle.c) so that a plan mistake in either one shows up
as a log L mismatch in tests/test_oracle_pins.py. Feasible up to a few thousand points.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg
import scipy.stats

E_OVER_100 = math.e / 100.0     # PAPER.md:135, default offset


def cov(d, cov_kind, sigma2, rho):
    """Exponential or Matern-3/2 (BASELINE C2, reading R3)."""
    if cov_kind == 0:
        return sigma2 * np.exp(-d / rho)
    a = math.sqrt(3.0) * d / rho
    return sigma2 * (1.0 + a) * np.exp(-a)


def dist(ax, ay, bx, by, xs=1.0, ys=1.0):
    dx = (np.asarray(ax)[:, None] - np.asarray(bx)[None, :]) * xs
    dy = (np.asarray(ay)[:, None] - np.asarray(by)[None, :]) * ys
    return np.sqrt(dx * dx + dy * dy)


class Tree:
    """Multi-resolution partition + knots."""

    def __init__(self, x, y, M, J, r, offset=E_OVER_100):
        assert J in (2, 4) and M >= 1 and r >= 1
        self.M, self.J, self.r, self.offset = M, J, r, offset
        self.nx = math.isqrt(r - 1) + 1 if r > 1 else 1      # ceil(sqrt r)
        self.ny = r // self.nx                               # floor(r / ceil(sqrt r))
        self.rh = self.nx * self.ny
        x0, x1, y0, y1 = float(np.min(x)), float(np.max(x)), float(np.min(y)), float(np.max(y))
        # data domain with top and right boundaries pushed out 1%
        root = (x0, x1 + 0.01 * (x1 - x0), y0, y1 + 0.01 * (y1 - y0))
        self.boxes = {(1, 0): root}
        for m in range(1, M):
            for t in range(J ** (m - 1)):
                bx0, bx1, by0, by1 = self.boxes[(m, t)]
                mx, my = 0.5 * (bx0 + bx1), 0.5 * (by0 + by1)
                if J == 4:   # SW, SE, NW, NE
                    kids = [(bx0, mx, by0, my), (mx, bx1, by0, my), (bx0, mx, my, by1), (mx, bx1, my, by1)]
                elif (bx1 - bx0) >= (by1 - by0):   # longer axis; tie -> x
                    kids = [(bx0, mx, by0, by1), (mx, bx1, by0, by1)]
                else:
                    kids = [(bx0, bx1, by0, my), (bx0, bx1, my, by1)]
                for c, b in enumerate(kids):
                    self.boxes[(m + 1, t * J + c)] = b

    def bars(self, lo, hi, nb):
        if nb == 1:
            return [0.5 * (lo + hi)]
        ext = hi - lo
        return [lo + self.offset * ext + i * (ext * (1.0 - 2.0 * self.offset) / (nb - 1)) for i in range(nb)]

    def knots(self, m, t):
        bx0, bx1, by0, by1 = self.boxes[(m, t)]
        xb = self.bars(bx0, bx1, self.nx)
        yb = self.bars(by0, by1, self.ny)
        kx = np.array([xb[ix] for iy in range(self.ny) for ix in range(self.nx)])
        ky = np.array([yb[iy] for iy in range(self.ny) for ix in range(self.nx)])
        return kx, ky

    def region_at(self, px, py, m):
        """Index (within level m) of the region containing (px, py): half-open boxes."""
        for t in range(self.J ** (m - 1)):
            bx0, bx1, by0, by1 = self.boxes[(m, t)]
            if bx0 <= px < bx1 and by0 <= py < by1:
                return t
        raise ValueError("point outside the root domain")

    def leaf_of(self, x, y):
        """Leaf index per observation, -1 if it coincides with a pre-finest knot."""
        knots = set()
        for m in range(1, self.M):
            for t in range(self.J ** (m - 1)):
                kx, ky = self.knots(m, t)
                knots.update(zip(kx.tolist(), ky.tolist()))
        out = np.empty(len(x), dtype=np.int64)
        for i, (px, py) in enumerate(zip(x, y)):
            out[i] = -1 if (float(px), float(py)) in knots else self.region_at(px, py, self.M)
        return out


def sigma_mra(x, y, M, J, r, cov_kind, sigma2, rho, offset=E_OVER_100, xs=1.0, ys=1.0,
              return_all=False, qx=None, qy=None):
    """Sigma_MRA over the retained observations (and optionally over Z = obs ∪ knots ∪ queries).

    Query points (prediction locations) join Z as finest-level points: the recursion is applied
    to every pair of points exactly as to the observations, so Sigma_MRA(q, s) is the MRA
    covariance the approximation assigns to a pair (q, s) (identical to C for same-leaf pairs)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    tree = Tree(x, y, M, J, r, offset)
    leaf = tree.leaf_of(x, y)
    keep = np.nonzero(leaf >= 0)[0]
    zx, zy = list(x[keep]), list(y[keep])
    nq = 0 if qx is None else len(qx)
    if nq:
        zx.extend(np.asarray(qx, dtype=np.float64).tolist())
        zy.extend(np.asarray(qy, dtype=np.float64).tolist())
    knot_sets = {}
    for m in range(1, M):
        for t in range(J ** (m - 1)):
            kx, ky = tree.knots(m, t)
            knot_sets[(m, t)] = list(range(len(zx), len(zx) + len(kx)))
            zx.extend(kx.tolist()); zy.extend(ky.tolist())
    zx, zy = np.array(zx), np.array(zy)
    nz = len(zx)
    reg = np.array([[tree.region_at(zx[i], zy[i], m) for m in range(1, M + 1)] for i in range(nz)])
    Cm = cov(dist(zx, zy, zx, zy, xs, ys), cov_kind, sigma2, rho)
    Sig = np.zeros((nz, nz))
    for m in range(1, M):
        T = np.zeros((nz, nz))
        for t in range(J ** (m - 1)):
            mem = np.nonzero(reg[:, m - 1] == t)[0]
            Q = np.array(knot_sets[(m, t)])
            if mem.size == 0:
                continue
            CQQ = Cm[np.ix_(Q, Q)]
            CaQ = Cm[np.ix_(mem, Q)]
            T[np.ix_(mem, mem)] = CaQ @ np.linalg.solve(CQQ, CaQ.T)
        Sig += T
        same = reg[:, m][:, None] == reg[:, m][None, :]
        Cm = np.where(same, Cm - T, 0.0)
    Sig += Cm
    nobs = keep.size
    if return_all:
        return Sig, keep, nobs, knot_sets, tree
    return Sig[:nobs, :nobs], keep


def loglik(x, y, z, M, J, r, cov_kind, sigma2, rho, tau2, **kw):
    """log N(z; 0, Sigma_MRA + tau2 I) by scipy (the exact Gaussian log-density)."""
    S, keep = sigma_mra(x, y, M, J, r, cov_kind, sigma2, rho, **kw)
    C = S + tau2 * np.eye(S.shape[0])
    return float(scipy.stats.multivariate_normal(mean=np.zeros(S.shape[0]), cov=C).logpdf(np.asarray(z)[keep]))


def logdet_quad(x, y, z, M, J, r, cov_kind, sigma2, rho, tau2, **kw):
    S, keep = sigma_mra(x, y, M, J, r, cov_kind, sigma2, rho, **kw)
    C = S + tau2 * np.eye(S.shape[0])
    sign, ld = np.linalg.slogdet(C)
    zz = np.asarray(z)[keep]
    return float(ld), float(zz @ scipy.linalg.solve(C, zz, assume_a="pos"))


def exact_gp_loglik(x, y, z, cov_kind, sigma2, rho, tau2):
    """Full (un-approximated) GP log-likelihood: the M=1 special case."""
    C = cov(dist(x, y, x, y), cov_kind, sigma2, rho) + tau2 * np.eye(len(x))
    return float(scipy.stats.multivariate_normal(mean=np.zeros(len(x)), cov=C).logpdf(z))


def posterior(x, y, z, M, J, r, cov_kind, sigma2, rho, tau2, **kw):
    """E[X(s)|y] at the observations and at every knot: Sigma[., obs] (Sigma_MRA + tau2 I)^{-1} y."""
    Sig, keep, nobs, knot_sets, tree = sigma_mra(x, y, M, J, r, cov_kind, sigma2, rho, return_all=True, **kw)
    C = Sig[:nobs, :nobs] + tau2 * np.eye(nobs)
    alpha = scipy.linalg.solve(C, np.asarray(z)[keep], assume_a="pos")
    ez = Sig[:, :nobs] @ alpha
    smooth = np.full(len(x), np.nan)
    smooth[keep] = ez[:nobs]
    xq = {k: ez[np.array(v)] for k, v in knot_sets.items()}
    return smooth, xq


def predict(x, y, z, qx, qy, M, J, r, cov_kind, sigma2, rho, tau2, **kw):
    """Conditional mean / variance of the noise-free X at query points under the MRA prior (the
    DEFINITION: kriging with Sigma_MRA): mean = Sigma(q, S) (Sigma(S,S) + tau2 I)^{-1} y,
    var = Sigma(q,q) - Sigma(q,S) (Sigma(S,S) + tau2 I)^{-1} Sigma(S,q)."""
    Sig, keep, nobs, knot_sets, tree = sigma_mra(x, y, M, J, r, cov_kind, sigma2, rho, return_all=True,
                                                 qx=qx, qy=qy, **kw)
    nq = len(qx)
    qi = np.arange(nobs, nobs + nq)
    C = Sig[:nobs, :nobs] + tau2 * np.eye(nobs)
    Sqs = Sig[np.ix_(qi, np.arange(nobs))]
    alpha = scipy.linalg.solve(C, np.asarray(z)[keep], assume_a="pos")
    mean = Sqs @ alpha
    var = np.diag(Sig[np.ix_(qi, qi)]) - np.einsum("ij,ji->i", Sqs, scipy.linalg.solve(C, Sqs.T, assume_a="pos"))
    return mean, var
