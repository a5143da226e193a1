"""Two-stream timeline of one pipelined step, eager: filter bank of batch i on
stream F, detect / describe / match of batch i-1 on stream X, CUDA events at
the stage boundaries (ms from the common start), and each half alone."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_00319_b200 import BatchPipeline, RiftConfig, engine, synth  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 16
imgs, _ = synth.make_batch(P, 1024, seed0=0)
pipe = BatchPipeline(P, 1024, 1024, RiftConfig(scale_mult=1.6, sigma_on_f=0.75))
pipe.load(imgs)
pipe.capture()
f2 = {k: torch.zeros_like(v) for k, v in pipe.f.items()}
pipe.run_fields(pipe.images, f2, "p_")
torch.cuda.synchronize()
SF, SX = torch.cuda.Stream(), torch.cuda.Stream()
c = pipe.cfg


def ev():
    return torch.cuda.Event(enable_timing=True)


def step(do_f=True, do_x=True):
    e0 = ev()
    e0.record()
    SF.wait_event(e0)
    SX.wait_event(e0)
    ef, ex = [ev()], [ev(), ev(), ev()]
    with torch.cuda.stream(SX):
        if do_x:
            engine.detect(f2["mmin"], f2["mmax"], c.fast_threshold, pipe.K, c.patch_size // 2, ws_key="tl_detect",
                          out=pipe.k, moment_range=f2["range"])
        ex[0].record(SX)
        if do_x:
            engine.describe(f2["mim"], pipe.k["x"], pipe.k["y"], pipe.k["count"], c.n_orient, c.patch_size, c.grid,
                            c.dominant_ratio, c.rotate_patch, pipe.desc_mode, capacity=pipe.cap,
                            ws_key="tl_describe", out=pipe.d)
        ex[1].record(SX)
        if do_x:
            engine.match(pipe.d, pipe.dim, pipe.rb, pipe.tb, pipe.K, ws_key="tl_match", out=pipe.m)
        ex[2].record(SX)
    with torch.cuda.stream(SF):
        if do_f:
            engine.fields(pipe.images, pipe.bank, out=pipe.f, ws_key="tl_fields")
        ef[0].record(SF)
    torch.cuda.current_stream().wait_stream(SF)
    torch.cuda.current_stream().wait_stream(SX)
    torch.cuda.synchronize()
    t = lambda e: round(e0.elapsed_time(e), 3)  # noqa: E731
    return {"fields_end": t(ef[0]), "detect_end": t(ex[0]), "describe_end": t(ex[1]), "match_end": t(ex[2])}


for _ in range(3):
    step()
res = {"both": [step() for _ in range(5)][-1], "fields_alone": step(True, False), "features_alone": step(False, True)}
print(json.dumps(res))
