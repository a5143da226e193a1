"""Time the match stage and the GEMM for the bench batch under different column splits (env R2_GEMM_SPLITS)."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2303_00319_b200 import BatchPipeline, RiftConfig, synth, engine
imgs, _ = synth.make_batch(16, 1024, seed0=0)
pipe = BatchPipeline(16, 1024, 1024, RiftConfig(max_keypoints=5000, scale_mult=1.6, sigma_on_f=0.75))
pipe.load(imgs); pipe.step(); torch.cuda.synchronize()
ms = bench.graph_ms(lambda: engine.match(pipe.d, pipe.dim, pipe.rb, pipe.tb, pipe.K, ws_key="x", out=pipe.m), 20)
dcnt = pipe.d["count"].cpu().numpy().astype(np.int64)
fl = float(sum(2 * dcnt[2 * q] * dcnt[2 * q + 1] * 216 for q in range(16)))
print(json.dumps({"splits": os.environ.get("R2_GEMM_SPLITS"), "match_ms": ms, "tflops": fl / ms / 1e9}))
