"""Device vs host time of the BASELINE generator's target side (warp,
inversion, gamma, speckle, renormalisation) for a batch of 1024^2 pairs.

PYTHONPATH=. python tools/synth_timing.py [--pairs 16] [--looks 4]
"""
import argparse
import json
import time

import numpy as np
import torch

from paper_2303_00319_b200 import engine, synth

ap = argparse.ArgumentParser()
ap.add_argument("--pairs", type=int, default=16)
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--looks", type=int, default=4)
args = ap.parse_args()
P, N = args.pairs, args.size
src = np.stack([synth.blob_field(N, i) for i in range(2)] * (P // 2))
params = np.zeros((P, 8))
for i in range(P):
    tr, _ = synth._pair_draws(N, i, None, 0.1, args.looks)
    params[i, :6] = synth.inverse_map(tr.matrix).ravel()
    params[i, 6:] = (tr.gamma, (1 if tr.inverted else 0) | 2)
d_src = torch.from_numpy(src).cuda()
d_par = torch.from_numpy(params).cuda()
d_looks = torch.full((P,), args.looks, dtype=torch.int32, device="cuda")
out = torch.empty((2 * P, N, N), dtype=torch.float32, device="cuda")
for _ in range(3):
    engine.synth_targets(d_src, d_par, d_looks, 1, out[1::2], src_copy=out[0::2])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    engine.synth_targets(d_src, d_par, d_looks, 1, out[1::2], src_copy=out[0::2])
e1.record()
torch.cuda.synchronize()
dev_ms = e0.elapsed_time(e1) / reps
# host: the same target side for one pair (warp + radiometry + numpy gamma speckle)
t0 = time.perf_counter()
img1, tr = src[0], synth._pair_draws(N, 0, None, 0.1, args.looks)[0]
v = synth.warp(img1, tr.matrix)
v = np.clip(1.0 - v, 0.0, 1.0) ** tr.gamma
if args.looks:
    v = v * np.random.default_rng(0).gamma(float(args.looks), 1.0 / args.looks, v.shape)
v = (v - v.min()) / max(v.max() - v.min(), 1e-12)
host_ms = (time.perf_counter() - t0) * 1e3
traffic = P * N * N * (8 + 8 + 8 + 4 + 4)
print(json.dumps(dict(pairs=P, size=N, looks=args.looks, device_ms_per_batch=dev_ms,
                      device_targets_per_s=P / dev_ms * 1e3, host_ms_per_target=host_ms,
                      host_targets_per_s=1e3 / host_ms, algorithmic_GBps=traffic / dev_ms / 1e6)))
