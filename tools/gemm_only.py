"""k_match_gemm alone (rift2_match_partial, graph-replayed) on the bench's 16-pair batch:
burst (one launch after an idle gap, median) and back-to-back ms, and TFLOP/s."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2303_00319_b200 import BatchPipeline, RiftConfig, engine, synth  # noqa: E402

imgs, _ = synth.make_batch(16, 1024, seed0=0)
pipe = BatchPipeline(16, 1024, 1024, RiftConfig(max_keypoints=5000, scale_mult=1.6, sigma_on_f=0.75))
pipe.load(imgs)
pipe.step()
torch.cuda.synchronize()
parts = engine.match_partial(pipe.d, pipe.dim, pipe.rb, pipe.tb)
f = lambda: engine.match_partial(pipe.d, pipe.dim, pipe.rb, pipe.tb, out=parts)  # noqa: E731
b2b = bench.graph_ms(f, 20)
burst = bench.graph_ms(f, 20, gap_s=0.02)
d = pipe.d["count"].cpu().numpy().astype(np.int64)
fl = float(sum(2 * d[2 * q] * d[2 * q + 1] * 216 for q in range(16)))
print(json.dumps({"burst_ms": burst, "b2b_ms": b2b, "burst_tflops": fl / burst / 1e9, "frac_burst": fl / burst / 1e9 / 1651.3}))
