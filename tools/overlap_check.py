"""Step time: overlapped two-stream step graph vs the sequential graphs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_00319_b200 import BatchPipeline, RiftConfig, synth  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 16
imgs, _ = synth.make_batch(P, 1024, seed0=0)
pipe = BatchPipeline(P, 1024, 1024, RiftConfig(scale_mult=1.6, sigma_on_f=0.75))
pipe.load(imgs)
pipe.capture()


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def seq():
    pipe.replay_fields()
    pipe.replay_features()


print(f"{P} pairs: overlapped step {timeit(pipe.step):.3f} ms, sequential {timeit(seq):.3f} ms, "
      f"fields alone {timeit(pipe.replay_fields):.3f} ms, features alone {timeit(pipe.replay_features):.3f} ms")

pipe.capture_pipelined()
pipe._alt.copy_(pipe.images)
state = {"i": 0}


def piped():
    pipe.pipelined_step(state["i"] & 1)
    state["i"] += 1


print(f"{P} pairs: pipelined step {timeit(piped):.3f} ms")
# results of the pipelined path equal the plain step's
pipe.step()
torch.cuda.synchronize()
want = {k: v.clone() for k, v in pipe.m.items()}
piped()
piped()
torch.cuda.synchronize()
same = all(torch.equal(want[k], pipe.m[k]) for k in want)
print("pipelined matches equal plain step:", same)
