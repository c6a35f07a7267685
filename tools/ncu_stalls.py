"""Summarise an `ncu --set full` report: speed-of-light lines, pipe / issue metrics and the warp-stall breakdown
(PC-sampling counts and shares), plus the top stalled SASS instructions. Usage: ncu_stalls.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys


def ncu(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep):
    rows = ncu(rep, "--page", "details", "--csv")
    h = rows[0]
    keep = ("Duration", "DRAM Throughput", "Compute (SM) Throughput", "L2 Hit Rate", "Issue Slots Busy",
            "Executed Ipc Active", "No Eligible", "Warp Cycles Per Issued Instruction", "Achieved Occupancy",
            "Registers Per Thread")
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in keep:
            print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
    raw = ncu(rep, "--page", "raw", "--csv")
    d = dict(zip(raw[0], raw[2] if len(raw) > 2 else raw[1]))
    for k in ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
              "dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k in d:
            print(f"{k:40s} {d[k]}")
    pre = "smsp__pcsamp_warps_issue_stalled_"
    st = {k[len(pre):]: float(v) for k, v in d.items() if k.startswith(pre) and not k.endswith("_not_issued")
          and v.replace(".", "", 1).isdigit()}
    tot = sum(st.values())
    print("warp stall samples (all), share:")
    for k, v in sorted(st.items(), key=lambda t: -t[1])[:12]:
        print(f"  {k:32s} {v:12.0f} {100 * v / max(tot, 1):5.1f}%")
    sass = ncu(rep, "--page", "source", "--csv", "--print-source", "sass")
    hh = sass[1]
    ia, isrc, iss = hh.index("Address"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
    items = []
    for r in sass[2:]:
        if len(r) < len(hh):
            continue
        try:
            items.append((float(r[iss]), r[ia], r[isrc]))
        except ValueError:
            pass
    tot = sum(x[0] for x in items)
    print("top stalled instructions of the kernel body (share of its samples):")
    for v, a, src in sorted(items, reverse=True)[:10]:
        print(f"  {100 * v / max(tot, 1):5.1f}% {a[-6:]} {src[:80]}")


if __name__ == "__main__":
    main(sys.argv[1])
