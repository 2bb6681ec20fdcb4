"""Summarise ncu reports / launch lists (run in the dev container on pulled gpurun_out files)."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "launch__grid_size", "smsp__average_warp_latency_issue_stalled_long_scoreboard"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summary(rep):
    h, u, data = raw(rep)
    for r in data:
        name = r[h.index("Kernel Name")].split("(")[0]
        print(f"--- {name}")
        for k in KEYS:
            if k in h:
                print(f"   {k:66s} {r[h.index(k)]:>16s} {u[h.index(k)]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", ""))
        v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:50s} launches={n:4d} ms={t:9.3f} share={100 * t / tot:5.1f}%")
    print(f"total ms {tot:.3f} over {sum(n for n, _ in agg.values())} launches")


if __name__ == "__main__":
    for a in sys.argv[1:]:
        (launches if a.endswith(".csv") else summary)(a)
