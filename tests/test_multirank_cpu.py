"""Multi-rank (world_size 2 and 3, gloo, CPU) test of the subtree-sharding path:
shard ownership from the product's host plan partitions the shard level exactly, and merging the
sum-reduced exchange buffer on rank 0 reproduces the single-process log-likelihood."""
import json
import os
import socket
import subprocess
import sys

import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,case", [(2, (6000, 5, 4, 9, 11, 3)), (3, (4000, 7, 2, 6, 12, 0)),
                                        (2, (5000, 4, 2, 16, 13, 2))])
def test_sharded_exchange_matches_single_process(world, case):
    from paper_1905_00141_b200 import build
    build.build()
    port = _free_port()
    procs = []
    for rank in range(world):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), OMP_NUM_THREADS="1")
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "_multirank_worker.py")]
                                      + [str(v) for v in case], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
    res = json.loads(outs[0][0].strip().splitlines()[-1])
    assert res["owned_counts"] == [1] * len(res["owned_counts"])     # every shard owned exactly once
    n, M, J, r, seed, cl = case
    x, y, z = synth.uniform_small(n, seed=seed, clusters=cl)
    single = oracle.run(x, y, z, M, J, r, (0, 1.0, 0.1, 0.05))["loglik"]
    assert abs(res["loglik"] - single) <= 1e-12 * abs(single)
