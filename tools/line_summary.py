"""Per-source-line instruction counts from `ncu --page source --csv --print-source cuda,sass`."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fname = "?"
hdr = None
cur_line = None
agg = collections.Counter()
stall = collections.Counter()
text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0].isdigit():
        cur_line = (fname, int(r[0]))
        text[cur_line] = r[1].strip()[:90]
    ie = r[hdr["Instructions Executed"]] if len(r) > hdr["Instructions Executed"] else ""
    if ie.isdigit() and cur_line:
        agg[cur_line] += int(ie)
        s = r[hdr["Warp Stall Sampling (All Samples)"]]
        stall[cur_line] += int(s) if s.isdigit() else 0
tot = sum(agg.values())
tst = sum(stall.values()) or 1
print("total warp instructions", tot)
for k, n in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    print(f"{100 * n / tot:5.1f}% inst {100 * stall[k] / tst:5.1f}% stall  {k[0]}:{k[1]}  {text.get(k, '')}")
