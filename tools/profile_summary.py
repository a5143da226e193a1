"""Summarise an ncu launch list of `bench.py` into profiles/.

usage: python tools/profile_summary.py LAUNCHES.csv OUT_PREFIX [steps]

LAUNCHES.csv is `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --clock-control none --csv` of a bench command.  Writes
OUT_PREFIX.txt (per-kernel table: launches, mean us, share of our kernel
time, DRAM bytes per launch) and OUT_PREFIX.json (the same, plus the
filter-bank DRAM traffic per step that bench.py reports as roofline.traffic).
ncu times are cold-cache and serialised: compare shares, not absolutes.
"""

import collections
import csv
import json
import re
import sys

FIELDS_KERNELS = ("k_rows_fwd", "k_cols", "k_rows_amp0", "k_rows_amp0_tma", "k_med_bins", "k_med_collect", "k_med_h2", "k_med_h3", "k_med_final", "k_rows_pc_tma",
                  "k_rows_pc")


def short(name: str) -> str:
    m = re.search(r"(k_[A-Za-z0-9_]+)", name)
    return m.group(1) if m else name.split("(")[0][:40]


def main():
    path, prefix = sys.argv[1], sys.argv[2]
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = {h: i for i, h in enumerate(rows[0])}
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        lid = int(r[hdr["ID"]])
        names[lid] = r[hdr["Kernel Name"]]
        v = r[hdr["Metric Value"]].replace(",", "")
        per[lid][r[hdr["Metric Name"]]] = float(v) if v else 0.0
    agg = collections.OrderedDict()
    for lid in sorted(per):
        k = short(names[lid])
        if not k.startswith("k_"):
            continue                                  # torch fill/copy kernels are not ours
        a = agg.setdefault(k, dict(n=0, ns=0.0, rd=0.0, wr=0.0))
        a["n"] += 1
        a["ns"] += per[lid].get("gpu__time_duration.sum", 0.0)
        a["rd"] += per[lid].get("dram__bytes_read.sum", 0.0)
        a["wr"] += per[lid].get("dram__bytes_write.sum", 0.0)
    tot = sum(a["ns"] for a in agg.values())
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else max(a["n"] for a in agg.values())
    lines = [f"# {path}: {sum(a['n'] for a in agg.values())} launches of our kernels, "
             f"{steps} pipeline passes; ncu gpu__time_duration (cold, serialised)",
             f"{'kernel':24s} {'launches':>8s} {'mean us':>9s} {'share':>6s} {'DRAM rd MB':>11s} {'DRAM wr MB':>11s}"]
    out = {"source": path, "passes": steps, "kernels": {}}
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        n = a["n"]
        lines.append(f"{k:24s} {n:8d} {a['ns'] / n / 1e3:9.1f} {a['ns'] / tot:6.1%} "
                     f"{a['rd'] / n / 1e6:11.1f} {a['wr'] / n / 1e6:11.1f}")
        out["kernels"][k] = {"launches": n, "mean_us": a["ns"] / n / 1e3, "share": a["ns"] / tot,
                             "dram_read_bytes_per_launch": a["rd"] / n, "dram_write_bytes_per_launch": a["wr"] / n}
    fb = [k for k in agg if k in FIELDS_KERNELS]
    fb_bytes = sum((agg[k]["rd"] + agg[k]["wr"]) / agg[k]["n"] * (agg[k]["n"] / steps) for k in fb)
    fb_ns = sum(agg[k]["ns"] for k in fb) / steps
    out["filter_bank"] = {"kernels": fb, "dram_bytes_per_pass": fb_bytes, "ncu_us_per_pass": fb_ns / 1e3,
                          "share_of_our_kernel_time": sum(agg[k]["ns"] for k in fb) / tot}
    lines.append(f"filter bank: {fb_bytes / 1e9:.2f} GB DRAM per pass, {fb_ns / 1e6:.3f} ms per pass (ncu), "
                 f"{out['filter_bank']['share_of_our_kernel_time']:.1%} of our kernel time")
    open(prefix + ".txt", "w").write("\n".join(lines) + "\n")
    json.dump(out, open(prefix + ".json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
