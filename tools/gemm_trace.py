"""Per-tile pipeline trace of k_match_gemm CTA (0,0) (needs the R2_GEMM_TRACE build)."""
import ctypes
import os
import sys

import numpy as np

os.environ["RIFT2_B200_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                            "paper_2303_00319_b200", "_libtrace", "librift2_b200.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_00319_b200 import _lib, engine  # noqa: E402

rng = np.random.default_rng(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 9000
P = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cap = n
counts = torch.zeros((2 * P, cap, 224), dtype=torch.float16)
counts[:, :, :216] = torch.from_numpy(rng.integers(0, 20, (2 * P, cap, 216)).astype(np.float16))
sq = (counts.float() ** 2).sum(-1).int()
kp = torch.arange(cap, dtype=torch.int32).repeat(2 * P, 1) // 2
desc = dict(counts=counts.cuda(), sqnorm=sq.cuda(), kp=kp.cuda(), count=torch.full((2 * P,), n, dtype=torch.int32).cuda())
rb = torch.arange(0, 2 * P, 2, dtype=torch.int32).cuda()
tb = rb + 1
for it in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    engine.match(desc, 216, rb, tb, cap)
    e.record()
    torch.cuda.synchronize()
    print(f"match {P} pairs of {n}x{n}: {s.elapsed_time(e):.3f} ms")
lib = _lib.load()
buf = (ctypes.c_ulonglong * (8 * 512))()
lib.rift2_debug_gemm_trace.restype = ctypes.c_int
lib.rift2_debug_gemm_trace(buf)
t = np.frombuffer(buf, dtype=np.uint64).reshape(8, 512).astype(np.int64)
t0 = t[0, 0]
names = ["prod pre-empty", "prod got-empty", "mma pre-full", "mma got-full", "mma got-tempty", "mma committed",
         "epi pre-tfull", "epi got-tfull"]
nt = int((t[5] > 0).sum())
lo, hi = min(8, nt // 4), nt
print("tiles traced", nt)
for i in list(range(0, 6)) + list(range(max(6, nt - 4), nt)):
    print(i, " ".join(f"{n[:14]}={(t[k, i] - t0) if t[k, i] else -1:>8d}" for k, n in enumerate(names)))
d = np.diff(t[5, lo:hi])
print("mma commit interval cycles: median", np.median(d), "mean", d.mean())
print("mma wait full  (cyc): median", np.median(t[3, lo:hi] - t[2, lo:hi]))
print("mma wait tempty(cyc): median", np.median(t[4, lo:hi] - t[3, lo:hi]))
print("epi wait tfull (cyc): median", np.median(t[7, lo:hi] - t[6, lo:hi]))
print("epi tile interval   : median", np.median(np.diff(t[7, lo:hi])))
print("prod wait empty(cyc): median", np.median(t[1, lo:hi] - t[0, lo:hi]))
