"""Streamed prior rows: a plan whose prior chain rows of the
levels >= the chunk level are computed per chunk of subtrees, right before that chunk's posterior pass,
instead of being resident for the whole tree. Every region's arithmetic is unchanged, so log L and the
per-region terms must equal the resident plan's bitwise and the oracle's within the north_star tolerance.
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


@pytest.mark.parametrize("n,M,J,r,cov,cl,wide", [(8000, 5, 4, 16, EXP, 2, 0), (8000, 5, 4, 16, EXP, 2, -1),
                                                 (6000, 7, 2, 25, MAT, 3, 0), (12800, 5, 4, 64, EXP, 3, 0)])
def test_streamed_prior_matches_resident_and_oracle(mra, n, M, J, r, cov, cl, wide):
    x, y, z = synth.uniform_small(n, seed=31 + M, clusters=cl)
    theta = (cov, 1.0, 0.1, 0.05)
    res = mra.mra_plan_create(x, y, M, J, r, wide=wide, stream_prior=-1)
    stm = mra.mra_plan_create(x, y, M, J, r, wide=wide, stream_prior=1, mem_budget_gb=0.004)
    info_r, info_s = mra.mra_plan_memory(res), mra.mra_plan_memory(stm)
    assert not info_r["streams_prior"] and info_s["streams_prior"]
    n_c = J ** (info_s["chunk_level"] - 1)
    assert info_s["chunk_regions"] < n_c          # several chunks, so several prior passes
    a = mra.mra_loglik(res, z, theta, regions=True)
    b = mra.mra_loglik(stm, z, theta, regions=True)
    assert a["loglik"] == b["loglik"]             # identical per-region arithmetic and reduction order
    np.testing.assert_array_equal(a["region_d"], b["region_d"])
    np.testing.assert_array_equal(a["region_u"], b["region_u"])
    ref = oracle.run(x, y, z, M, J, r, theta)
    assert abs(b["loglik"] - ref["loglik"]) <= 1e-9 * abs(ref["loglik"])


def test_streamed_prior_auto_and_memory(mra):
    """Auto mode streams when the resident rows would take more than half the budget; the streaming
    plan holds less device memory than the resident one for the same budget."""
    x, y, z = synth.uniform_small(20000, seed=5, clusters=0)
    M, J, r = 6, 4, 64          # resident prior: 341 regions x m r^2 doubles ~ 44 MB
    res = mra.mra_plan_create(x, y, M, J, r, stream_prior=-1, mem_budget_gb=0.06)
    auto = mra.mra_plan_create(x, y, M, J, r, stream_prior=0, mem_budget_gb=0.06)
    assert not mra.mra_plan_memory(res)["streams_prior"]
    ia = mra.mra_plan_memory(auto)
    assert ia["streams_prior"]
    theta = (EXP, 1.0, 0.1, 0.05)
    assert mra.mra_loglik(res, z, theta)["loglik"] == mra.mra_loglik(auto, z, theta)["loglik"]
    big = mra.mra_plan_create(x, y, M, J, r, stream_prior=0)   # default budget: everything resident
    assert not mra.mra_plan_memory(big)["streams_prior"]


def test_streamed_prior_sharded_and_optimize(mra):
    """Sharded evaluation (ranks emulated in sequence on one GPU) and the optimizer on streaming plans."""
    import torch
    x, y, z = synth.uniform_small(12000, seed=10, clusters=3)
    theta = (EXP, 1.0, 0.1, 0.05)
    single = mra.mra_loglik(mra.mra_plan_create(x, y, 5, 4, 16, stream_prior=-1), z, theta)["loglik"]
    zd = torch.from_numpy(z).cuda()
    world = 3
    plans = [mra.mra_plan_create(x, y, 5, 4, 16, rank=k, world=world, stream_prior=1, mem_budget_gb=0.003)
             for k in range(world)]
    assert all(mra.mra_plan_memory(p)["streams_prior"] for p in plans)
    size = mra.mra_shard_size(plans[0])
    total = torch.zeros(size, dtype=torch.float64, device="cuda")
    for pl in plans:
        buf = torch.zeros(size, dtype=torch.float64, device="cuda")
        mra.mra_loglik_shard(pl, zd, theta, buf)
        total += buf
    ll = mra.mra_loglik_finish(plans[0], theta, total)
    assert abs(ll - single) <= 1e-12 * abs(single)
    p_res = mra.mra_plan_create(x, y, 5, 4, 16, stream_prior=-1)
    p_stm = mra.mra_plan_create(x, y, 5, 4, 16, stream_prior=1, mem_budget_gb=0.003)
    o1 = mra.mra_optimize(p_res, zd, theta, max_evals=12)
    o2 = mra.mra_optimize(p_stm, zd, theta, max_evals=12)
    assert o1[1] == o2[1] and tuple(o1[0]) == tuple(o2[0]) and o1[2] == o2[2]


def test_streamed_prior_refuses_posterior_state(mra):
    x, y, z = synth.uniform_small(3000, seed=3)
    p = mra.mra_plan_create(x, y, 4, 4, 16, stream_prior=1)
    theta = (EXP, 1.0, 0.1, 0.05)
    assert np.isfinite(mra.mra_loglik(p, z, theta)["loglik"])
    with pytest.raises(mra.MraError) as e:
        mra.mra_loglik(p, z, theta, posterior=True)
    assert e.value.status == 2
    with pytest.raises(mra.MraError):
        mra.mra_predict(p, x[:10], y[:10])
