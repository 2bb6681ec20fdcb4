"""Per-opcode and per-region histogram of an ncu source page (SASS):
    ncu -i REP --page source --csv --print-source sass > src.csv
    python profiles/sass_hist.py src.csv
Prints warp-level executed instructions by opcode, stall samples by opcode, and
the hottest address ranges, to see where a kernel's issue slots go."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc, iex, ismp = (h.index("Address"), h.index("Source"), h.index("Instructions Executed"),
                       h.index("Warp Stall Sampling (All Samples)"))
ops = collections.Counter()
smp = collections.Counter()
tot = 0
seq = []
for r in rows[2:]:
    if len(r) <= iex or not r[iex].isdigit():
        continue
    src = r[isrc].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    n = int(r[iex])
    ops[op] += n
    smp[op] += int(r[ismp] or 0)
    tot += n
    seq.append((r[ia], src, n, int(r[ismp] or 0)))
print(f"total warp instructions executed: {tot}")
for op, n in ops.most_common(40):
    print(f"  {op:12s} {n:12d} {100 * n / tot:6.2f}%   stall samples {smp[op]}")
if len(sys.argv) > 2:
    for a, s, n, sm in seq:
        print(f"{a[-5:]} {n:9d} {sm:6d}  {s}")
