"""Pipelined step (fields of batch i || features of batch i-1) launched
eagerly on two streams, with and without a high-priority features stream,
and as graphs captured on priority streams, vs the plain graph step."""
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
pipe.capture_pipelined()
pipe._alt.copy_(pipe.images)
fbuf = (pipe.f, pipe._f2)
ibuf = (pipe.images, pipe._alt)


def timeit(fn, n=20):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        fn(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print(f"graph pipelined: {timeit(lambda i: pipe.pipelined_step(i & 1)):.3f} ms")
for lo_p, hi_p in ((0, 0), (0, -1), (-1, 0)):
    s_fields = torch.cuda.Stream(priority=lo_p)
    s_feat = torch.cuda.Stream(priority=hi_p)

    def step(i):
        p = i & 1
        cur = torch.cuda.current_stream()
        s_feat.wait_stream(cur)
        s_fields.wait_stream(cur)
        with torch.cuda.stream(s_feat):
            pipe.run_features(fbuf[1 - p], "p_")
        with torch.cuda.stream(s_fields):
            pipe.run_fields(ibuf[p], fbuf[p], "p_")
        cur.wait_stream(s_feat)
        cur.wait_stream(s_fields)

    print(f"eager pipelined, fields prio {lo_p}, features prio {hi_p}: {timeit(step):.3f} ms")

    g = [torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()]
    cap = torch.cuda.Stream(priority=lo_p)
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap):
        for p in (0, 1):
            with torch.cuda.graph(g[p], stream=cap):
                s_feat.wait_stream(cap)
                with torch.cuda.stream(s_feat):
                    pipe.run_features(fbuf[1 - p], "p_")
                pipe.run_fields(ibuf[p], fbuf[p], "p_")
                cap.wait_stream(s_feat)
    torch.cuda.synchronize()
    print(f"graph pipelined, fields prio {lo_p}, features prio {hi_p}: {timeit(lambda i: g[i & 1].replay()):.3f} ms")
