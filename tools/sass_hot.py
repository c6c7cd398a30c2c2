"""Aggregate an ncu --page source --csv (SASS) dump: warp-instructions and
stall samples per opcode, and the hottest instructions (tools only)."""
import collections
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
r = list(csv.reader(l for l in open(path) if not l.startswith("==")))
hdr = r[1]
rows = [dict(zip(hdr, x)) for x in r[2:] if len(x) == len(hdr)]
num = lambda s: float(s.replace(",", "")) if s not in ("", "-") else 0.0
by_op = collections.defaultdict(lambda: [0.0, 0.0])
tot_i = tot_s = 0.0
for d in rows:
    src = d["Source"].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    i, s = num(d["Instructions Executed"]), num(d["Warp Stall Sampling (All Samples)"])
    by_op[op][0] += i
    by_op[op][1] += s
    tot_i += i
    tot_s += s
print(f"total warp-instructions {tot_i:.4g}, samples {tot_s:.4g}")
for op, (i, s) in sorted(by_op.items(), key=lambda x: -x[1][0])[:top]:
    print(f"  {op:12s} inst {i:12.4g} ({100*i/tot_i:5.1f}%)  samples {100*s/tot_s:5.1f}%")
print("hottest instructions by samples:")
for d in sorted(rows, key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))[:top]:
    print(f"  {d['Address'][-5:]} {num(d['Warp Stall Sampling (All Samples)']):6.0f} {d['Source'].strip()[:90]}")
