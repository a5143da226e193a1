"""Debug: self-pair matching on the reference CLI test's voronoi image."""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
from rift2.synthetic import voronoi_label_map
import rift2
import paper_2303_00319_b200 as r2
img = voronoi_label_map(256, 40, seed=12)
for kp in (200, 150):
    cfg = r2.RiftConfig(max_keypoints=kp)
    res = r2.match_pair(img, img, cfg)
    d = np.array([p[2] for p in res.matches.pairs])
    print("max_kp", kp, "n", len(d), "nonzero", int((d != 0).sum()), d[d != 0][:5])
    # reference matcher on our descriptors
    ref = [rift2.descriptor.Descriptor(x.vector, x.keypoint_id, x.variant, x.mode) for x in res.ref.descriptors]
    tgt = [rift2.descriptor.Descriptor(x.vector, x.keypoint_id, x.variant, x.mode) for x in res.tgt.descriptors]
    want = rift2.match_nn(ref, tgt)
    print("  ref matcher nonzero", sum(1 for p in want.pairs if p[2] != 0), "same set", {(a, b) for a, b, _ in want.pairs} == {(a, b) for a, b, _ in res.matches.pairs})
    bad = [(a, b, c) for a, b, c in res.matches.pairs if c != 0][:5]
    for a, b, c in bad:
        ra = [x for x in res.ref.descriptors if x.keypoint_id == a]
        tb = [x for x in res.tgt.descriptors if x.keypoint_id == b]
        rb = [x for x in res.ref.descriptors if x.keypoint_id == b]
        print("  pair", a, b, c, "ref variants", [x.variant for x in ra], "tgt variants", [x.variant for x in tb],
              "self variants", [x.variant for x in rb],
              "cos(best)", max(float(np.dot(x.vector, y.vector)) for x in ra for y in tb),
              "cos(self)", max(float(np.dot(x.vector, y.vector)) for x in rb for y in tb))
    w = {b: (a, c) for a, b, c in want.pairs}
    for a, b, c in bad[:3]:
        print("  ref says", b, "->", w.get(b))
