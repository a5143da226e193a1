"""HBM read-only / write-only / copy bandwidth with torch kernels (CUDA events).
python tools/hbm_rw.py -> one JSON line (GB/s, bytes moved / time)."""
import json

import torch


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


n = 1 << 30   # 4 GiB of fp32
x = torch.empty(n, device="cuda")
y = torch.empty(n, device="cuda")
x.fill_(1.0)
out = {}
out["write_fill"] = 4 * n / t(lambda: x.fill_(2.0)) / 1e6
out["read_sum"] = 4 * n / t(lambda: x.sum()) / 1e6
out["read_amax"] = 4 * n / t(lambda: x.amax()) / 1e6
out["copy_rw"] = 8 * n / t(lambda: y.copy_(x)) / 1e6
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
