import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import torch
import paper_2303_00319_b200 as r2
from paper_2303_00319_b200 import synth
cfg = r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75, max_keypoints=20000)
for kw in (dict(looks=None, radiometric=False), dict(looks=None), dict()):
    for size in (1024, 4096):
        a, b, truth = synth.make_pair(size, seed=2, **kw)
        t0 = time.time()
        res = r2.match_pair(a, b, cfg)
        torch.cuda.synchronize()
        dt = time.time() - t0
        rx = np.array([[k.x, k.y] for k in res.ref.keypoints]); tx = np.array([[k.x, k.y] for k in res.tgt.keypoints])
        r = np.array([p[0] for p in res.matches.pairs]); t = np.array([p[1] for p in res.matches.pairs])
        resid = np.linalg.norm(truth.apply(rx[r]) - tx[t], axis=1)
        print(size, kw, "kp", len(rx), len(tx), "matches", len(r), "correct(<3px)", int((resid < 3).sum()), f"{dt:.2f}s")
