"""CUDA-event time of the filter bank alone (development tool).

python tools/fields_timing.py [--size 1024] [--pairs 16] [--iters 20]
Prints ms per pass and the fraction of the HBM roofline (429 B/px/image).
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_00319_b200 import RiftConfig, engine, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--pairs", type=int, default=16)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    imgs, _ = synth.make_batch(min(args.pairs, 2), args.size, looks=4)
    reps = (args.pairs + 1) // 2
    imgs = np.concatenate([imgs] * reps)[: 2 * args.pairs]
    x = torch.as_tensor(imgs).cuda()
    bank = RiftConfig(scale_mult=1.6, sigma_on_f=0.75).bank_params()
    for _ in range(3):
        f = engine.fields(x, bank)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.iters)]
    for a, b in ev:
        a.record()
        engine.fields(x, bank, out=f)
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in ev)
    ms = float(np.median(ts))
    peak = 6547.8
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        pass
    byts = 429 * args.size * args.size * 2 * args.pairs
    print(json.dumps({"size": args.size, "pairs": args.pairs, "ms_median": ms, "ms_min": ts[0],
                      "GBps": byts / ms / 1e6, "frac": byts / ms / 1e6 / peak}))


if __name__ == "__main__":
    main()
