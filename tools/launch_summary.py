"""Summarise an ncu launch-list CSV (per kernel: launches, device ms, DRAM GB, DMMA-active %)."""
import collections
import csv
import sys


def load(path):
    hdr, by = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = by.setdefault(d["ID"], {"name": d["Kernel Name"]})
            try:
                e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
            except ValueError:
                pass
    return list(by.values())


def main(path, evals=1):
    rows = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for v in rows:
        a = agg[v["name"].split("(")[0][:48]]
        t = v.get("gpu__time_duration.sum", 0.0)
        a[0] += 1
        a[1] += t
        a[2] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
        a[3] += t * v.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
    tot = sum(a[1] for a in agg.values())
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:50s} n={a[0]:5d} ms/eval={a[1] / 1e6 / evals:9.2f} share={100 * a[1] / tot:5.1f}% "
              f"dram GB/eval={a[2] / 1e9 / evals:8.1f} dmma%={a[3] / max(a[1], 1):5.1f}")
    print(f"total ms/eval {tot / 1e6 / evals:.1f}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
