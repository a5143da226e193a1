"""Summarise an ncu source-page (SASS) CSV: instruction mix, stall samples, smem conflicts."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ops = collections.Counter()
stalls = collections.Counter()
excess = collections.Counter()
tot_inst = 0
tot_samp = 0
top = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[ix["Instructions Executed"]].isdigit():
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    base = op.split(".")[0]
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    e = int(r[ix["L1 Wavefronts Shared Excessive"]] or 0)
    ops[base] += n
    stalls[base] += s
    excess[base] += e
    tot_inst += n
    tot_samp += s
    top.append((s, src[:70], n, e))
print(f"warp instructions executed: {tot_inst}, stall samples: {tot_samp}")
print("opcode        inst%   stall%   smem-excess-wavefronts")
for op, n in ops.most_common(25):
    print(f"{op:12s} {100 * n / tot_inst:6.1f} {100 * stalls[op] / max(tot_samp, 1):7.1f}   {excess[op]}")
print("top stalled instructions:")
for s, src, n, e in sorted(top, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{s:7d} {n:9d} {e:8d}  {src}")
