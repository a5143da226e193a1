"""Per-CTA timeline of k_match_gemm in the 16-pair pipeline (needs the R2_GEMM_TRACE build)."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["RIFT2_B200_LIB"] = os.path.join(ROOT, "paper_2303_00319_b200", "_libtrace", "librift2_b200.so")
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2303_00319_b200 import BatchPipeline, RiftConfig, _lib, synth  # noqa: E402

imgs, _ = synth.make_batch(16, 1024, seed0=0)
pipe = BatchPipeline(16, 1024, 1024, RiftConfig(scale_mult=1.6, sigma_on_f=0.75))
pipe.load(imgs)
pipe.run()
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * (8192 * 4))()
lib.rift2_debug_gemm_ctas.restype = ctypes.c_int
lib.rift2_debug_gemm_ctas(buf)
c = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 4).astype(np.int64)
c = c[c[:, 1] > 0]
t0 = c[:, 1].min()
start, end, tiles, sm = (c[:, 1] - t0) / 1e3, (c[:, 2] - t0) / 1e3, c[:, 3], c[:, 0]
dur = end - start
act = tiles > 0
print(f"CTAs {len(c)}, active {act.sum()}, kernel span {end.max():.1f} us")
print(f"active CTA duration us: min {dur[act].min():.1f} median {np.median(dur[act]):.1f} max {dur[act].max():.1f}")
print(f"idle CTA duration us: median {np.median(dur[~act]):.2f}" if (~act).any() else "")
print("tiles per active CTA: min", tiles[act].min(), "median", np.median(tiles[act]), "max", tiles[act].max())
per_sm = np.zeros(160)
for s_, d_ in zip(sm, dur):
    per_sm[s_] += d_
print(f"busy us per SM: min {per_sm[:148].min():.1f} median {np.median(per_sm[:148]):.1f} max {per_sm[:148].max():.1f}")
order = np.argsort(start)
q = np.linspace(0, len(order) - 1, 9).astype(int)
print("start times (us) at deciles of launch order:", [round(float(start[order[i]]), 1) for i in q])
print("last 5 finishing CTAs: (start, end, tiles)", [(round(float(start[i]), 1), round(float(end[i]), 1), int(tiles[i])) for i in np.argsort(end)[-5:]])
