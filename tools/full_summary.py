"""Summarise one `ncu --set full --import-source on` capture for profiles/.

usage: python tools/full_summary.py REPORT.ncu-rep [KERNEL_REGEX] > profiles/rNN_full_<kernel>.txt

Prints the kernel's headline metrics, occupancy limits, warp-stall reasons
(per issued instruction), pipe utilisation and the source lines with the
most executed instructions.
"""

import csv
import io
import subprocess
import sys

REP = sys.argv[1]
KRE = sys.argv[2] if len(sys.argv) > 2 else None


def ncu(*args):
    cmd = ["ncu", "-i", REP, *args, "--csv"]
    if KRE:
        cmd[3:3] = ["-k", f"regex:{KRE}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


details = ncu("--page", "details")
h = details[0]
name = None
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Shared Memory Configuration Size",
        "Block Limit Registers", "Block Limit Shared Mem", "Theoretical Occupancy", "Achieved Occupancy"]
got = {}
for r in details[1:]:
    d = dict(zip(h, r))
    name = d.get("Kernel Name", name)
    m = d.get("Metric Name")
    if m in want and m not in got:
        got[m] = f"{d.get('Metric Value')} {d.get('Metric Unit')}"
print(name)
for m in want:
    if m in got:
        print(f"  {m:34s} {got[m]}")

raw = ncu("--page", "raw")
rh, rv = raw[0], dict(zip(raw[0], raw[2]))
stalls = []
for k in rh:
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            stalls.append((float(rv[k]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
print("warp stalls per issued instruction (top 8):")
for v, k in sorted(stalls, reverse=True)[:8]:
    print(f"  {k:24s} {v:6.2f}")
pipes = []
for k in rh:
    if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active"):
        try:
            pipes.append((float(rv[k]), k[len("sm__inst_executed_pipe_"):-len(".avg.pct_of_peak_sustained_active")]))
        except ValueError:
            pass
for k in ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"):
    if k in rv:
        print(f"  {k:72s} {rv[k]}")
print("pipe utilisation, % of peak (top 6):")
for v, k in sorted(pipes, reverse=True)[:6]:
    print(f"  {k:24s} {v:6.1f}")

src = ncu("--page", "source", "--print-source", "cuda,sass")
agg, text, hdr, cur, fname = {}, {}, None, None, "?"
for r in src:
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
        text[cur] = r[1].strip()[:80]
    ie = r[hdr["Instructions Executed"]] if len(r) > hdr["Instructions Executed"] else ""
    if ie.isdigit() and cur:
        agg[cur] = agg.get(cur, 0) + int(ie)
tot = sum(agg.values()) or 1
print("source lines by executed instructions (top 12):")
for k, n in sorted(agg.items(), key=lambda kv: -kv[1])[:12]:
    print(f"  {100 * n / tot:5.1f}%  {k[0]}:{k[1]}  {text.get(k, '')}")
