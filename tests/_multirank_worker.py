"""Worker for tests/test_multirank_cpu.py (one process per rank, gloo backend, CPU only).

Each rank asks the product's host-side plan (device = -2, no GPU) which level-s shards it owns
(LPT assignment), evaluates those subtrees with the oracle, writes their outputs
into its slots of a zero-initialised exchange buffer, and the buffers are sum-reduced to rank 0
(the collective the GPU path issues through NCCL); rank 0 merges the levels above s."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import paper_1905_00141_b200 as mra  # noqa: E402
import synth  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    n, M, J, r, seed, cl = (int(v) for v in sys.argv[1:7])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, y, z = synth.uniform_small(n, seed=seed, clusters=cl)
    theta = (0, 1.0, 0.1, 0.05)
    plan = mra.mra_plan_create(x, y, M, J, r, device=-2, rank=rank, world=world)
    sh = mra.mra_plan_shards(plan)
    s = sh["shard_level"]
    ns = J ** (s - 1)
    P = (s - 1) * plan.r_hat
    per = P * P + P + 2
    buf = torch.zeros(ns * per, dtype=torch.float64)
    for t in sh["own"].tolist():
        o = oracle.run(x, y, z, M, J, r, theta, target=(s, t), outputs=True, nthreads=1)
        blk = np.concatenate([o["A"].ravel(), o["omega"], [o["d"], o["u"]]])
        buf[t * per:(t + 1) * per] = torch.from_numpy(blk)
    dist.reduce(buf, dst=0, op=dist.ReduceOp.SUM)
    owned = torch.zeros(ns, dtype=torch.int64)
    owned[torch.from_numpy(sh["own"])] = 1
    dist.reduce(owned, dst=0, op=dist.ReduceOp.SUM)
    if rank == 0:
        b = buf.numpy().reshape(ns, per)
        ll = oracle.finish(x, y, z, M, J, r, theta, s, b[:, :P * P].reshape(ns, P, P), b[:, P * P:P * P + P],
                           b[:, -2], b[:, -1])
        print(json.dumps({"loglik": ll, "shard_level": s, "owned_counts": owned.tolist(),
                          "own0": sh["own"].tolist()}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
