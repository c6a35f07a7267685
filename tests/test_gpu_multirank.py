"""The PRODUCT's multi-GPU path end to end in separate processes, compared with the ORACLE.

(1) two / three OS processes (one per rank) each run the sm_100a shard pass of its own subtrees
    (mra_loglik_shard_post), the exchange buffers are sum-reduced to rank 0 (gloo), rank 0 merges the levels
    above the shard level (mra_loglik_finish_post), the above-shard means are broadcast and every rank
    finishes its own posterior (mra_posterior_shard). All ranks share cuda:0 (this box has one GPU); no
    kernel waits on another rank's kernel -- the only coupling is the host-side collective between passes.
(2) the in-library exchange (opts.nccl_id: ncclBroadcast of the above-shard prior rows, ncclReduce of the
    packed exchange buffer, ncclBroadcast of log L and the above-shard means, ncclAllReduce of the posterior
    outputs) at world 1 -- NCCL does not allow two ranks on one device, so the 2..8-rank case is covered by
    the same code at world 1 here plus the gloo test above.
Tolerances (north_star): log L relative 1e-9, posterior means / smoothing normwise 1e-8."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _post_close(mu_g, mu_r, sm_g, sm_r, tol=1e-8):
    assert np.max(np.abs(mu_g - mu_r)) <= tol * np.max(np.abs(mu_r))
    assert np.array_equal(np.isnan(sm_g), np.isnan(sm_r))
    assert np.nanmax(np.abs(sm_g - sm_r)) <= tol * np.nanmax(np.abs(sm_r))


@pytest.mark.parametrize("world,case", [(2, (6000, 5, 4, 16, 11, 3, 0)), (3, (5000, 7, 2, 9, 12, 0, 1)),
                                        (2, (20000, 5, 4, 36, 13, 2, 0))])
def test_product_shards_in_separate_processes_vs_oracle(mra, world, case, tmp_path):
    port = _free_port()
    out = tmp_path / "rank0.json"
    procs = []
    for rank in range(world):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), OMP_NUM_THREADS="1")
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "_multirank_gpu_worker.py")]
                                      + [str(v) for v in case] + [str(out)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=900) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-3000:]
    res = json.loads(out.read_text())
    assert res["mu_owners_max"] <= 1.0 and res["smooth_owners_max"] <= 1.0   # each entry from one rank
    n, M, J, r, seed, cl, cov = case
    x, y, z = synth.uniform_small(n, seed=seed, clusters=cl)
    theta = (cov, 1.0, 0.1, 0.05)
    ref = oracle.run(x, y, z, M, J, r, theta, posterior=True)
    assert abs(res["loglik"] - ref["loglik"]) <= 1e-9 * abs(ref["loglik"])
    _post_close(np.array(res["mu"]), ref["mu"].ravel(), np.array(res["smooth"]), ref["smooth"])


NCCL_CASES = [(4000, 4, 4, 16, 21, 0, 0), (5000, 6, 2, 30, 22, 3, 1), (12000, 5, 4, 64, 23, 2, 0)]


@pytest.mark.parametrize("case", NCCL_CASES)
def test_in_library_nccl_exchange_vs_oracle(mra, case):
    import torch
    n, M, J, r, seed, cl, cov = case
    x, y, z = synth.uniform_small(n, seed=seed, clusters=cl)
    theta = (cov, 1.0, 0.1, 0.05)
    p = mra.mra_plan_create(x, y, M, J, r, device=0, nccl_id=mra.mra_nccl_unique_id(), rank=0, world=1,
                            stream=torch.cuda.current_stream())
    assert mra.mra_plan_shards(p)["shard_level"] >= 2
    got = mra.mra_loglik(p, z, theta, posterior=True, regions=True)
    ref = oracle.run(x, y, z, M, J, r, theta, posterior=True, regions=True)
    assert abs(got["loglik"] - ref["loglik"]) <= 1e-9 * abs(ref["loglik"])
    ok = ~np.isnan(ref["region_d"])
    assert np.all(np.abs(got["region_d"][ok] - ref["region_d"][ok]) <= 1e-8 * np.maximum(1, np.abs(ref["region_d"][ok])))
    assert np.all(np.abs(got["region_u"][ok] - ref["region_u"][ok]) <= 1e-8 * np.maximum(1, np.abs(ref["region_u"][ok])))
    _post_close(got["mu"].ravel(), ref["mu"].ravel(), got["smooth"], ref["smooth"])
    # prediction through the broadcast above-shard factors equals the oracle's recursion
    rng = np.random.default_rng(seed)
    qx, qy = rng.random(300), rng.random(300)
    qx[:3] = [-1.0, 0.5, 2.0]
    mean, var = mra.mra_predict(p, qx, qy)
    rm, rv = oracle.predict(x, y, z, qx, qy, M, J, r, theta)
    assert np.array_equal(np.isnan(mean), np.isnan(rm))
    assert np.nanmax(np.abs(mean - rm)) <= 1e-8 * np.nanmax(np.abs(rm))
    assert np.nanmax(np.abs(var - rv)) <= 1e-8 * np.nanmax(np.abs(rv))
    # device-y entry: same kernels and the same collectives -> bitwise the host-y value
    zd = torch.from_numpy(z).cuda()
    assert mra.mra_loglik_dev(p, zd, theta)["loglik"] == got["loglik"]
    p.close()


def test_in_library_nccl_sweep_and_optimizer(mra):
    """theta sweeps and the optimizer run collectively on a communicator plan (every rank sees the
    broadcast log L, so every rank takes the same search steps)."""
    import torch
    x, y, z = synth.uniform_small(3000, seed=31)
    p = mra.mra_plan_create(x, y, 4, 4, 16, device=0, nccl_id=mra.mra_nccl_unique_id(), rank=0, world=1)
    q = mra.mra_plan_create(x, y, 4, 4, 16, device=0)
    zd = torch.from_numpy(z).cuda()
    ths = [(0, 1.0, rho, 0.05) for rho in (0.05, 0.1, 0.2)]
    a = mra.mra_loglik_batch_dev(p, zd, ths)
    b = mra.mra_loglik_batch_dev(q, zd, ths)
    assert np.all(np.abs(a - b) <= 1e-11 * np.abs(b))
    th, ll, ne = mra.mra_optimize(p, zd, (0, 1.0, 0.1, 0.05), lower=(0.1, 0.01, 0.001), upper=(10, 1, 1),
                                  max_evals=60)
    th2, ll2, ne2 = mra.mra_optimize(q, zd, (0, 1.0, 0.1, 0.05), lower=(0.1, 0.01, 0.001), upper=(10, 1, 1),
                                     max_evals=60)
    assert ne > 4 and abs(ll - ll2) <= 1e-7 * abs(ll2)          # same search up to rounding-order ties


def test_torch_allocator_hooks_bitwise(mra):
    """opts.dalloc / dfree (torch's caching allocator): the same plan arithmetic, bitwise the same result,
    and the plan's memory shows up in torch's allocator statistics."""
    import torch
    x, y, z = synth.uniform_small(6000, seed=41, clusters=2)
    theta = (0, 1.0, 0.1, 0.05)
    before = torch.cuda.memory_allocated()
    p = mra.mra_plan_create(x, y, 5, 4, 16, device=0, torch_alloc=True, stream=torch.cuda.current_stream())
    assert torch.cuda.memory_allocated() - before >= mra.mra_plan_memory(p)["device_bytes"] // 2
    q = mra.mra_plan_create(x, y, 5, 4, 16, device=0, stream=torch.cuda.current_stream())
    a = mra.mra_loglik(p, z, theta, posterior=True)
    b = mra.mra_loglik(q, z, theta, posterior=True)
    assert a["loglik"] == b["loglik"]
    assert np.array_equal(a["smooth"], b["smooth"], equal_nan=True)
    m1, v1 = mra.mra_predict(p, x[:50], y[:50])
    m2, v2 = mra.mra_predict(q, x[:50], y[:50])
    assert np.array_equal(m1, m2) and np.array_equal(v1, v2)
    p.close()
    q.close()
