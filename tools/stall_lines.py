"""Source lines ranked by one warp-stall reason, from `ncu --page source --csv --print-source cuda,sass`.

usage: python tools/stall_lines.py SOURCE.csv [stall_long_sb] [N]
"""
import csv
import sys

path = sys.argv[1]
key = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
hdr, cur, fname = None, None, "?"
agg, text = {}, {}
for r in csv.reader(open(path, errors="replace")):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {x: i for i, x in enumerate(r)}
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0].isdigit():
        cur = (fname, int(r[0]))
        text[cur] = r[1].strip()[:90]
    v = r[hdr[key]] if len(r) > hdr[key] else ""
    if v.isdigit() and cur:
        agg[cur] = agg.get(cur, 0) + int(v)
tot = sum(agg.values()) or 1
for k, n in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * n / tot:5.1f}%  {k[0]}:{k[1]}  {text.get(k, '')}")
