"""Per-stage CUDA-event timing of the batched pipeline (development tool).

python tools/stage_timing.py [--size 1024] [--pairs 16] [--iters 5]
"""

import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_00319_b200 import RiftConfig, engine, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--pairs", type=int, default=16)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--max-kp", type=int, default=5000)
    args = ap.parse_args()
    t0 = time.time()
    imgs, _ = synth.make_batch(min(args.pairs, 4), args.size)
    reps = (args.pairs + 3) // 4
    imgs = np.concatenate([imgs] * reps)[: 2 * args.pairs]
    print(f"generated in {time.time() - t0:.1f}s", flush=True)
    x = torch.as_tensor(imgs).cuda()
    bank = RiftConfig(scale_mult=1.6, sigma_on_f=0.75).bank_params()
    B = x.shape[0]
    rb = torch.arange(0, B, 2, dtype=torch.int32, device="cuda")
    tb = rb + 1

    def run():
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        f = engine.fields(x, bank)
        ev[1].record()
        k = engine.detect(f["mmin"], f["mmax"], 0.001, args.max_kp, 48)
        ev[2].record()
        d = engine.describe(f["mim"], k["x"], k["y"], k["count"], 6, capacity=2 * args.max_kp)
        ev[3].record()
        m = engine.match(d, 216, rb, tb, args.max_kp)
        ev[4].record()
        torch.cuda.synchronize()
        return [ev[i].elapsed_time(ev[i + 1]) for i in range(4)], k, d, m

    for it in range(args.iters):
        ts, k, d, m = run()
        tot = sum(ts)
        print(f"iter {it}: fields {ts[0]:.2f} ms, detect {ts[1]:.2f}, describe {ts[2]:.2f}, "
              f"match {ts[3]:.2f}; total {tot:.2f} ms -> {args.pairs / tot * 1e3:.1f} pairs/s", flush=True)
    print("kp counts", k["count"].cpu().numpy()[:8], "desc counts", d["count"].cpu().numpy()[:8],
          "matches", m["count"].cpu().numpy()[:4])


if __name__ == "__main__":
    main()
