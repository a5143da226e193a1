"""cProfile of the dataclass API (match_pair) on one 1024^2 BASELINE pair."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_00319_b200 as r2  # noqa: E402
from paper_2303_00319_b200 import synth  # noqa: E402

cfg = r2.RiftConfig(scale_mult=1.6, sigma_on_f=0.75)
a, b, _ = synth.make_pair(1024, 0)
r2.match_pair(a, b, cfg)
t0 = time.perf_counter()
r2.match_pair(a, b, cfg)
print("wall", time.perf_counter() - t0)
pr = cProfile.Profile()
pr.enable()
r2.match_pair(a, b, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
