"""Full-size parity against the ORACLE's stored values (BASELINE.json configs C2, C3, C4 at their real sizes,
in the launch configuration bench.py times: one plan on cuda:0, default options).

The stored values (tests/golden/full_*.json / *_post.npz) were written by tools/make_golden.py, which calls
only oracle/ on the inputs synth generates on the CPU (bitwise reproducible across CPU instruction sets and
thread counts); each entry carries the SHA-256 of its input arrays, so a stale golden is reported as such,
not as a parity failure. Bars (north_star): log L relative 1e-9 (PAPER.md:84-97 recursion); every stored
region's d_R / u_R 1e-8 relative to max(1, |ref|) (basis invariant); posterior means and
smoothed values (C2) normwise 1e-8 (R12)."""
import glob
import hashlib
import json
import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


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


_W = {}


def _workload(name):
    if name not in _W:
        _W.clear()
        w = synth.make(name)           # CPU generation: the bits the golden was computed on
        h = hashlib.sha256()
        for a in (w.x, w.y, w.z):
            h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
        _W[name] = (w, h.hexdigest())
    return _W[name]


def _goldens(name):
    return sorted(glob.glob(os.path.join(GOLD, f"full_{name}*.json")))


def _check(mra, name, files, posterior=False):
    import torch
    if not files:
        pytest.skip(f"no golden for {name} (tools/make_golden.py)")
    w, sha = _workload(name)
    p = mra.mra_plan_create(w.x, w.y, w.M, w.J, w.r, stream=torch.cuda.current_stream())
    zd = torch.from_numpy(w.z).cuda()
    for fn in files:
        g = json.load(open(fn))
        assert g["input_sha256"] == sha, f"{fn}: stale golden (inputs changed)"
        theta = tuple(g["theta"])
        got = mra.mra_loglik_dev(p, zd, theta, regions=True, posterior=posterior)
        assert p.n_retained == g["n_retained"]
        rel = abs(got["loglik"] - g["loglik"]) / abs(g["loglik"])
        assert rel <= 1e-9, (fn, got["loglik"], g["loglik"], rel)
        for key, ref in (("region_d", g["region_d"]), ("region_u", g["region_u"])):
            ref = np.array(ref)
            gv = got[key][: ref.shape[0]]
            ok = ~np.isnan(ref)
            bad = np.abs(gv[ok] - ref[ok]) > 1e-8 * np.maximum(1, np.abs(ref[ok]))
            assert not bad.any(), (fn, key, np.max(np.abs(gv[ok] - ref[ok])))
        if posterior:
            post = np.load(os.path.join(GOLD, g["post_file"]))
            for key in ("region_d", "region_u"):
                ref = post[key]
                ok = ~np.isnan(ref)
                assert np.all(np.abs(got[key][ok] - ref[ok]) <= 1e-8 * np.maximum(1, np.abs(ref[ok]))), key
            mu = got["mu"].cpu().numpy().ravel()
            assert np.max(np.abs(mu - post["mu"].ravel())) <= 1e-8 * g["mu_absmax"]
            sm = got["smooth"].cpu().numpy()[post["smooth_idx"]]
            ref = post["smooth"]
            assert np.array_equal(np.isnan(sm), np.isnan(ref))
            assert np.nanmax(np.abs(sm - ref)) <= 1e-8 * g["smooth_absmax"]
    p.close()


def test_C2_full_loglik_regions_mu_smoothing(mra):
    """C2: 1,048,576 observations, Matern-3/2, M=8: log L, all 21,845 d_R / u_R, mu, smoothing."""
    _check(mra, "C2", _goldens("C2"), posterior=True)


def test_C3_full_47M_loglik(mra):
    """C3: the 47,000,000-observation headline workload: log L and the top-5-level d_R / u_R."""
    _check(mra, "C3", _goldens("C3"))


def test_C4_full_loglik_thetas(mra):
    """C4: 2,000,000 swath observations (leaves up to ~9k), every theta of the sweep with a golden."""
    _check(mra, "C4", _goldens("C4"))
