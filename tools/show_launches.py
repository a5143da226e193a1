"""Print per-kernel time / instructions / IPC / DRAM bytes from tools/launches.sh output."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import load  # noqa: E402

agg = load(sys.argv[1])
minus = float(sys.argv[2]) if len(sys.argv) > 2 else 100.0
tot = 0.0
for (i, k), v in sorted(agg.items()):
    t = v.get("gpu__time_duration.sum", 0)
    tot += t
    if t > minus * 1e3:
        inst = v.get("sm__inst_executed.sum", 0)
        name = k.split("(")[0].split("::")[-1] if "::" in k else k
        print(f"{name[:30]:30s} {t / 1e3:9.1f} us  inst {inst / 1e6:8.1f} M  warps {v.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):5.1f}%"
              f"  IPC/SM {inst / (t * 1.965) / 148:5.2f}  rd {v.get('dram__bytes_read.sum', 0) / 1e9:6.2f} GB"
              f"  wr {v.get('dram__bytes_write.sum', 0) / 1e9:6.2f} GB")
print(f"total {tot / 1e6:.3f} ms")
