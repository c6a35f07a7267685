"""Seeded synthetic inputs for the MRA log-likelihood hot path.

This module is shared by the oracle-side tests and the CUDA-side tests/bench. It
holds NO arithmetic of the MRA method (no partition, knots, recursion or
likelihood): only the data-generating processes that stand in for the paper's
MODIS/AMSR data (PAPER.md:372, 597, 764 -- not available here), as fixed by
BASELINE.json `configs` and the readings SURVEY.md §8(c) L19-L24 / DESIGN.md §3.

Configs (0-based):
  C0  4,096 U[0,1]^2, exp(s2=1, rho=0.1, tau2=0.05), y ~ exact dense GP + nugget, M=3 J=4 r=16
  C1  131,072 U[0,1]^2, exp(1, 0.05, 0.01), cosine field K=64 + N(0,0.01), M=6 J=4 r=36
  C2  1024^2 jittered grid on [0,360]x[-90,90], Matern-1.5(2, 5, 0.1), cosine K=64, M=8 J=4 r=64
  C3  47,000,000 U([0,360]x[-90,90]), exp(1, 2, 0.05), cosine K=256, M=10 J=4 r=64
  C4  2,000,000 in 40 parallel strips (width 0.02) over [0,1]^2, exp(1, rho, tau2) on a 4x4
      (rho, tau2) grid, cosine K=64, M=11 J=2 r=32 (r_hat=30)

Every config can be generated at a reduced `n` with the same recipe (same domain,
same field, same tree shape) for parity tests that the oracle finishes in seconds.
Seeds: config k uses seed k unless overridden.

The paper's binary data format ("u64 n, then n lon, n lat, n values,
all 64-bit reals") is provided by `write_paper_format` / `read_paper_format`.
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field

import numpy as np

COV_EXP = 0
COV_MATERN32 = 1


@dataclass
class Workload:
    name: str
    x: np.ndarray          # [n] fp64 longitude / x
    y: np.ndarray          # [n] fp64 latitude / y
    z: np.ndarray          # [n] fp64 observed values (the paper's "values")
    M: int
    J: int
    r: int
    thetas: list = field(default_factory=list)   # list of (cov, sigma2, rho, tau2)
    domain: tuple = (0.0, 1.0, 0.0, 1.0)
    recipe: str = ""

    @property
    def n(self) -> int:
        return int(self.x.shape[0])


# nominal parameters of BASELINE.json configs[0..4]
SPECS = {
    "C0": dict(n=4096, M=3, J=4, r=16, domain=(0.0, 1.0, 0.0, 1.0),
               thetas=[(COV_EXP, 1.0, 0.1, 0.05)]),
    "C1": dict(n=131072, M=6, J=4, r=36, domain=(0.0, 1.0, 0.0, 1.0),
               thetas=[(COV_EXP, 1.0, 0.05, 0.01)], modes=64),
    "C2": dict(n=1024 * 1024, M=8, J=4, r=64, domain=(0.0, 360.0, -90.0, 90.0),
               thetas=[(COV_MATERN32, 2.0, 5.0, 0.1)], modes=64),
    "C3": dict(n=47_000_000, M=10, J=4, r=64, domain=(0.0, 360.0, -90.0, 90.0),
               thetas=[(COV_EXP, 1.0, 2.0, 0.05)], modes=256),
    "C4": dict(n=2_000_000, M=11, J=2, r=32, domain=(0.0, 1.0, 0.0, 1.0),
               thetas=[(COV_EXP, 1.0, float(rho), float(t2))
                       for rho in np.linspace(0.02, 0.2, 4) for t2 in np.linspace(0.01, 0.2, 4)],
               modes=64, strips=40, width=0.02),
}


def _torch_device(device):
    if device is None:
        return None
    import torch
    return torch.device(device)


def cosine_field(xh: np.ndarray, yh: np.ndarray, modes: int, rng: np.random.Generator,
                 device=None, chunk: int = 1 << 22) -> np.ndarray:
    """f(s) = sum_i cos(2 pi k_i . s_hat + phi_i), s_hat in [0,1]^2.

    |k_i| ~ U(0, 20], direction ~ U[0, 2pi), phi_i ~ U[0, 2pi). Evaluated in fp64 with
    torch (on `device` if given, else CPU) in chunks; returns numpy fp64 f/std(f)."""
    mag = 20.0 * (1.0 - rng.random(modes))          # (0, 20]
    ang = 2.0 * math.pi * rng.random(modes)
    phi = 2.0 * math.pi * rng.random(modes)
    kx = 2.0 * math.pi * mag * np.cos(ang)
    ky = 2.0 * math.pi * mag * np.sin(ang)
    import torch
    dev = _torch_device(device) or torch.device("cpu")
    tkx = torch.tensor(kx, dtype=torch.float64, device=dev)
    tky = torch.tensor(ky, dtype=torch.float64, device=dev)
    tph = torch.tensor(phi, dtype=torch.float64, device=dev)
    n = xh.shape[0]
    out = np.empty(n, dtype=np.float64)
    step = max(1, chunk // max(1, modes // 16))
    for s in range(0, n, step):
        e = min(n, s + step)
        tx = torch.from_numpy(xh[s:e]).to(dev)
        ty = torch.from_numpy(yh[s:e]).to(dev)
        arg = tx[:, None] * tkx[None, :] + ty[:, None] * tky[None, :] + tph[None, :]
        out[s:e] = torch.cos(arg).sum(dim=1).cpu().numpy()
    sd = float(out.std())
    return out / sd


def _dense_gp_sample(x, y, sigma2, rho, tau2, rng):
    """C0's y: exact dense exponential GP + nugget, y = chol(C(S,S) + tau2 I) z.
    Data-generating process only (the method never forms this matrix)."""
    d = np.sqrt((x[:, None] - x[None, :]) ** 2 + (y[:, None] - y[None, :]) ** 2)
    c = sigma2 * np.exp(-d / rho)
    c[np.diag_indices_from(c)] += tau2
    L = np.linalg.cholesky(c)
    return L @ rng.standard_normal(x.shape[0])


def _strips(n: int, nstrips: int, width: float, rng: np.random.Generator):
    """C4 swaths (refined in DESIGN.md reading R11): `nstrips` parallel strips of
    `width` at one common random angle, offsets uniform over the projection range of the unit
    square. Points are uniform over the union of the strips clipped to [0,1]^2 (constant density
    along every swath, as in satellite swath data), so a strip gets a share of the n points
    proportional to its clipped area. Sampled by rejection in strip coordinates."""
    theta = math.pi * rng.random()
    t = np.array([math.cos(theta), math.sin(theta)])        # along-strip direction
    nrm = np.array([-t[1], t[0]])                           # across-strip normal
    corners = np.array([[0, 0], [1, 0], [0, 1], [1, 1]], dtype=np.float64)
    pn = corners @ nrm
    pt = corners @ t
    lo_n, hi_n = pn.min() + width / 2, pn.max() - width / 2
    offs = lo_n + (hi_n - lo_n) * rng.random(nstrips)
    tlo, thi = pt.min(), pt.max()

    def sample(o, m):
        u = tlo + (thi - tlo) * rng.random(m)
        v = o - width / 2 + width * rng.random(m)
        px = u * t[0] + v * nrm[0]
        py = u * t[1] + v * nrm[1]
        ok = (px >= 0) & (px < 1) & (py >= 0) & (py < 1)
        return px[ok], py[ok], ok.mean()

    # clipped area of each strip (Monte Carlo acceptance rate x bounding-rectangle area)
    area = np.array([sample(o, 20000)[2] for o in offs]) * (thi - tlo) * width
    share = area / area.sum()
    per = np.floor(share * n).astype(np.int64)
    per[: n - per.sum()] += 1
    xs, ys = [], []
    for o, cnt in zip(offs, per):
        got_x, got_y, have = [], [], 0
        while have < cnt:
            px, py, _ = sample(o, max(4 * (cnt - have), 1024))
            take = min(cnt - have, px.shape[0])
            got_x.append(px[:take]); got_y.append(py[:take]); have += take
        xs.append(np.concatenate(got_x)); ys.append(np.concatenate(got_y))
    return np.concatenate(xs), np.concatenate(ys)


def make(name: str, n: int | None = None, seed: int | None = None, device=None) -> Workload:
    """Generate config `name` (C0..C4), optionally at a reduced size `n` (same recipe)."""
    spec = SPECS[name]
    cfg_idx = int(name[1])
    seed = cfg_idx if seed is None else seed
    n = spec["n"] if n is None else int(n)
    rng = np.random.default_rng(seed)
    x0, x1, y0, y1 = spec["domain"]
    if name == "C2":
        side = int(round(math.sqrt(n)))
        if side * side != n:
            raise ValueError("C2 needs a square n (jittered side x side grid)")
        i = np.tile(np.arange(side, dtype=np.float64), side)
        j = np.repeat(np.arange(side, dtype=np.float64), side)
        x = (i + rng.random(n)) * (x1 - x0) / side + x0
        y = (j + rng.random(n)) * (y1 - y0) / side + y0
        recipe = f"jittered {side}x{side} grid on [0,360]x[-90,90] (SURVEY.md L22)"
    elif name == "C4":
        x, y = _strips(n, spec["strips"], spec["width"], rng)
        recipe = f"{spec['strips']} strips width {spec['width']}, uniform density over the swaths (DESIGN.md R11)"
    else:
        x = x0 + (x1 - x0) * rng.random(n)
        y = y0 + (y1 - y0) * rng.random(n)
        recipe = f"uniform on [{x0},{x1}]x[{y0},{y1}]"
    if name == "C0":
        cov, s2, rho, t2 = spec["thetas"][0]
        z = _dense_gp_sample(x, y, s2, rho, t2, rng)
        recipe += "; y = exact dense exponential GP + nugget (SURVEY.md L24)"
    else:
        xh = (x - x0) / (x1 - x0)
        yh = (y - y0) / (y1 - y0)
        f = cosine_field(xh, yh, spec["modes"], rng, device=device)
        z = f + 0.1 * rng.standard_normal(n)             # N(0, 0.01): variance 0.01 (L19)
        recipe += f"; y = cosine field K={spec['modes']} scaled to unit variance + N(0,0.01) (L20)"
    return Workload(name=name, x=np.ascontiguousarray(x), y=np.ascontiguousarray(y),
                    z=np.ascontiguousarray(z), M=spec["M"], J=spec["J"], r=spec["r"],
                    thetas=list(spec["thetas"]), domain=spec["domain"], recipe=recipe)


def uniform_small(n: int, seed: int, domain=(0.0, 1.0, 0.0, 1.0), clusters: int = 0):
    """Tiny random location sets for pins (optionally clustered so some leaves are empty).
    Returns (x, y, z) with z ~ N(0,1)."""
    rng = np.random.default_rng(seed)
    x0, x1, y0, y1 = domain
    if clusters:
        cx = rng.random(clusters); cy = rng.random(clusters)
        k = rng.integers(0, clusters, n)
        x = np.clip(cx[k] + 0.05 * rng.standard_normal(n), 0, 1)
        y = np.clip(cy[k] + 0.05 * rng.standard_normal(n), 0, 1)
    else:
        x = rng.random(n); y = rng.random(n)
    x = x0 + (x1 - x0) * x
    y = y0 + (y1 - y0) * y
    return x, y, rng.standard_normal(n)


def write_paper_format(path: str, x, y, z) -> None:
    """PAPER.md:172 binary layout: u64 n, n lon, n lat, n values (fp64, native little endian)."""
    n = int(len(x))
    with open(path, "wb") as f:
        f.write(struct.pack("<Q", n))
        for a in (x, y, z):
            f.write(np.ascontiguousarray(a, dtype="<f8").tobytes())


def read_paper_format(path: str):
    with open(path, "rb") as f:
        (n,) = struct.unpack("<Q", f.read(8))
        arr = np.frombuffer(f.read(24 * n), dtype="<f8")
    return arr[:n].copy(), arr[n:2 * n].copy(), arr[2 * n:].copy()
