"""Projected multi-GPU scaling from measured per-rank work, on ONE GPU (this pool has no multi-GPU node).

For world = 2, 4, 8 the config is planned once per rank exactly as each rank of `bench.py --gpus N` plans it (the
product's shard level and longest-processing-time assignment), each rank's shard pass (`mra_loglik_shard`: its
subtrees' prior, leaves and merges down to the shard level) is run and timed with CUDA events ALONE on the GPU, one
rank after another (no rank waits on another; nothing runs concurrently), the packed exchange buffers are summed on
the device (what ncclReduce does), and rank 0's finish (`mra_loglik_finish`: the merges above the shard level) is
timed. The projection of one N-GPU evaluation is

    max over ranks (shard pass)  +  finish  (+ the collectives: 9.6 MB reduce + a few KB of broadcasts at C3, not
                                             included -- tens of microseconds over NVLink 5)

Each rank's pass includes the above-shard prior levels that rank 0 computes and broadcasts in the in-library path
(every rank replicates them here). The result also checks that the summed exchange gives the single-GPU log L.
This is a projection from measured components, not a multi-GPU measurement.

Usage: python tools/project_scaling.py [--config C3] [--worlds 2,4,8] [--reps 2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1905_00141_b200 as mra  # noqa: E402
import synth  # noqa: E402


def timed(fn, reps):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    mra.load_library()
    w = synth.make(args.config, device="cuda")
    th = w.thetas[0]
    zd = torch.from_numpy(w.z).cuda()
    stream = torch.cuda.current_stream()
    p1 = mra.mra_plan_create(w.x, w.y, w.M, w.J, w.r, stream=stream)
    t1, ll1 = timed(lambda: mra.mra_loglik_dev(p1, zd, th)["loglik"], args.reps)
    n_ret = p1.n_retained
    p1.close()
    out = {"config": args.config, "n_retained": n_ret, "single_gpu_ms": t1, "single_gpu_loglik": ll1, "worlds": []}
    print(json.dumps({"single_gpu_ms": t1}), flush=True)
    for world in [int(v) for v in args.worlds.split(",")]:
        total = None
        rank_ms = []
        level = None
        # one plan alive at a time (a C3 plan holds most of the GPU); rank 0 last, it also runs the finish
        for rank in reversed(range(world)):
            p = mra.mra_plan_create(w.x, w.y, w.M, w.J, w.r, stream=stream, rank=rank, world=world)
            sh = mra.mra_plan_shards(p)
            level = sh["shard_level"]
            buf = torch.zeros(mra.mra_shard_size(p), dtype=torch.float64, device="cuda")
            ms, _ = timed(lambda: mra.mra_loglik_shard(p, zd, th, buf), args.reps)
            rank_ms.insert(0, ms)
            total = buf if total is None else total + buf
            if rank > 0:
                p.close()
                del p
        xmb = mra.mra_shard_size(p) * 8 / 1e6
        fin_ms, ll = timed(lambda: mra.mra_loglik_finish(p, th, total), args.reps)
        p.close()
        proj = max(rank_ms) + fin_ms
        row = {"world": world, "shard_level": level, "rank_ms": rank_ms, "finish_ms": fin_ms,
               "projected_ms": proj, "projected_obs_per_s": n_ret / (proj / 1e3), "speedup": t1 / proj,
               "efficiency": t1 / proj / world, "imbalance": max(rank_ms) / (sum(rank_ms) / world),
               "loglik": ll, "loglik_rel_vs_single": abs(ll - ll1) / abs(ll1),
               "exchange_mb": xmb}
        out["worlds"].append(row)
        print(json.dumps(row), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
