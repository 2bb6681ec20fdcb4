"""DRAM traffic per engine launch of each kernel class, from an ncu launch list
taken with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
over ONE epoch (bench.py, 1 GPU; with two or more optimizer steps in the list the
last complete epoch is used).  Kernels are assigned to the engine's classes
by name and by phase (forward = before k_loss_f32).  Writes profiles/ncu_traffic.json
{class: bytes per engine-level launch}, read by bench.py as roofline.traffic.

    python profiles/traffic_from_launches.py gpurun_out/traffic_rXX.csv [epoch_launch_counts.json]
"""
import collections
import csv
import json
import os
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
         "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
         "msecond": 1e-3}
# engine-level launches (kend calls) per class per epoch for the bench workload (P = 8, 3 layers)
# (one GPU: the forward GEMM runs once per partition over central + marginal rows for the
# aggregate-then-transform layers, twice for the transform-first one: 8 + 8 + 16)
KENDS = {"spmm_fwd": 48, "spmm_bwd": 16, "partials": 16, "quant": 40, "gemm_fwd": 32}


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, ni, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    idi = h.index("ID")
    launches = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[idi], {"name": r[ki].split("(")[0].replace("void ", "")})
        d[r[ni]] = float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0)
    seq = list(launches.values())
    adam = [i for i, d in enumerate(seq) if "k_adam" in d["name"]]
    if len(adam) >= 2:  # one whole epoch: after the penultimate optimizer step up to the last
        seq = seq[adam[-2] + 1:adam[-1] + 1]
    phase = "fwd"
    acc = collections.defaultdict(lambda: [0.0, 0.0])  # class -> [dram bytes, seconds]
    for d in seq:
        n = d["name"]
        if "k_loss_f32" in n:
            phase = "bwd"
        if "spmm" in n and phase == "fwd":
            cls = "spmm_fwd"
        elif "quantize_pack" in n:
            cls = "quant"
        elif "k_tc_gemm<0>" in n and phase == "fwd":
            cls = "gemm_fwd"
        else:
            continue
        acc[cls][0] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        acc[cls][1] += d.get("gpu__time_duration.sum", 0)
    out = {c: acc[c][0] / KENDS[c] for c in acc}
    dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
    json.dump(out, open(dst, "w"), indent=1)
    for c, (b, t) in acc.items():
        print(f"{c:10s} dram {b / 1e9:8.3f} GB/epoch  per launch {b / KENDS[c] / 1e6:9.1f} MB  "
              f"(ncu serialised time {t * 1e3:7.3f} ms, {b / t / 1e9 if t else 0:7.1f} GB/s)")


if __name__ == "__main__":
    main(sys.argv[1])
