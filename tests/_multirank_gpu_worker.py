"""Worker for tests/test_gpu_multirank.py: one process per rank, all on cuda:0, gloo for the collective.

Each rank builds the PRODUCT's sharded plan (rank, world, no in-library communicator), evaluates its own
subtrees with mra_loglik_shard_post (the sm_100a kernels), the exchange buffers are sum-reduced to rank 0
over gloo (host copies -- the collective the in-library path issues as ncclReduce), rank 0 merges the levels
above the shard level (mra_loglik_finish_post), the above-shard means are broadcast, and every rank finishes
its own posterior means / smoothed values (mra_posterior_shard). No rank's kernels wait on another rank's:
the only coupling is the host-side gloo collective between the two passes (tests/README: one GPU stands in
for the box). Rank 0 prints log L and the assembled posterior as JSON (file path in argv)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1905_00141_b200 as mra  # noqa: E402
import synth  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    n, M, J, r, seed, cl, cov = (int(v) for v in sys.argv[1:8])
    out_path = sys.argv[8]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    x, y, z = synth.uniform_small(n, seed=seed, clusters=cl)
    theta = (cov, 1.0, 0.1, 0.05)
    mra.load_library()
    plan = mra.mra_plan_create(x, y, M, J, r, device=0, rank=rank, world=world,
                               stream=torch.cuda.current_stream())
    zd = torch.from_numpy(z).cuda()
    size = mra.mra_shard_size(plan)
    buf = torch.zeros(size, dtype=torch.float64, device="cuda")
    mra.mra_loglik_shard_post(plan, zd, theta, buf)
    hb = buf.cpu()
    dist.reduce(hb, dst=0, op=dist.ReduceOp.SUM)
    mutop = torch.zeros(max(1, mra.mra_mutop_size(plan)), dtype=torch.float64, device="cuda")
    ll = float("nan")
    if rank == 0:
        ll = mra.mra_loglik_finish_post(plan, theta, hb.cuda(), mutop)
    ht = mutop.cpu()
    dist.broadcast(ht, src=0)
    mutop.copy_(ht)
    nmu = plan.n_interior * plan.r_hat
    dmu = torch.empty(max(1, nmu), dtype=torch.float64, device="cuda")
    dsm = torch.empty(n, dtype=torch.float64, device="cuda")
    mra.mra_posterior_shard(plan, mutop, dmu, dsm)
    torch.cuda.synchronize()
    mu = dmu.cpu()[:nmu]
    sm = dsm.cpu()
    # assemble: every entry is owned by exactly one rank (NaN elsewhere); the above-shard means are on all
    own_mu = (~torch.isnan(mu)).to(torch.float64)
    own_sm = (~torch.isnan(sm)).to(torch.float64)
    mu0, sm0 = torch.nan_to_num(mu), torch.nan_to_num(sm)
    s = mra.mra_plan_shards(plan)["shard_level"]
    top = (J ** (s - 1) - 1) // (J - 1) * plan.r_hat
    if rank != 0:                                  # count the replicated above-shard means once
        mu0[:top] = 0
        own_mu[:top] = 0
    for t in (mu0, sm0, own_mu, own_sm):
        dist.reduce(t, dst=0, op=dist.ReduceOp.SUM)
    if rank == 0:
        mu_full = torch.where(own_mu > 0, mu0, torch.full_like(mu0, float("nan")))
        sm_full = torch.where(own_sm > 0, sm0, torch.full_like(sm0, float("nan")))
        with open(out_path, "w") as f:
            json.dump({"loglik": ll, "shard_level": s, "mu": mu_full.tolist(), "smooth": sm_full.tolist(),
                       "mu_owners_max": float(own_mu.max()) if nmu else 1.0,
                       "smooth_owners_max": float(own_sm.max())}, f)
    plan.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
