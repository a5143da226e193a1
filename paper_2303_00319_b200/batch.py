"""Batched tensor API: the throughput path used by bench.py.

A BatchPipeline owns every device buffer for `n_pairs` image pairs of one
size (images interleaved [ref0, tgt0, ref1, tgt1, ...]) and runs the four
stages back to back on the current stream with no host synchronisation.
The two stage groups (filter bank; detect + describe + match) are captured
into CUDA graphs after a warm-up, so a step is two graph launches.
"""

from __future__ import annotations

import numpy as np
import torch

from . import engine
from .config import RiftConfig
from .errors import ParameterError


class BatchPipeline:
    def __init__(self, n_pairs: int, height: int, width: int, cfg: RiftConfig | None = None, device=None):
        self.cfg = cfg or RiftConfig()
        if self.cfg.mode != "rift2":
            raise ParameterError("the batched pipeline runs the rift2 mode")
        self.bank = self.cfg.bank_params()
        self.P, self.H, self.W = int(n_pairs), int(height), int(width)
        self.B = 2 * self.P
        self.K = int(self.cfg.max_keypoints)
        self.dev = torch.device(device or "cuda")
        B, H, W, K = self.B, self.H, self.W, self.K
        d = self.dev
        self.images = torch.zeros((B, H, W), dtype=torch.float32, device=d)
        self.f = dict(mmax=torch.empty((B, H, W), dtype=torch.float32, device=d),
                      mmin=torch.empty((B, H, W), dtype=torch.float32, device=d),
                      mim=torch.empty((B, H, W), dtype=torch.uint8, device=d))
        self.k = dict(x=torch.zeros((B, K), dtype=torch.int32, device=d),
                      y=torch.zeros((B, K), dtype=torch.int32, device=d),
                      response=torch.zeros((B, K), dtype=torch.float64, device=d),
                      kind=torch.zeros((B, K), dtype=torch.uint8, device=d),
                      count=torch.zeros((B,), dtype=torch.int32, device=d))
        cap = 2 * K
        self.d = dict(counts=torch.zeros((B, cap, engine.DESC_STRIDE), dtype=torch.float16, device=d),
                      sqnorm=torch.zeros((B, cap), dtype=torch.int32, device=d),
                      kp=torch.zeros((B, cap), dtype=torch.int32, device=d),
                      variant=torch.zeros((B, cap), dtype=torch.uint8, device=d),
                      count=torch.zeros((B,), dtype=torch.int32, device=d),
                      skipped=torch.zeros((B,), dtype=torch.int32, device=d))
        self.m = dict(ref=torch.zeros((self.P, K), dtype=torch.int32, device=d),
                      tgt=torch.zeros((self.P, K), dtype=torch.int32, device=d),
                      dist=torch.zeros((self.P, K), dtype=torch.float64, device=d),
                      count=torch.zeros((self.P,), dtype=torch.int32, device=d))
        self.rb = torch.arange(0, B, 2, dtype=torch.int32, device=d)
        self.tb = self.rb + 1
        self.dim = self.cfg.grid * self.cfg.grid * self.cfg.n_orient
        self.graphs = None
        self._alt = None
        self._copy_stream = None

    # ---- stages (eager) --------------------------------------------------
    def run_fields(self):
        engine.fields(self.images, self.bank, out=self.f, ws_key="b_fields")

    def run_features(self):
        c = self.cfg
        engine.detect(self.f["mmin"], self.f["mmax"], c.fast_threshold, self.K, c.patch_size // 2,
                      ws_key="b_detect", out=self.k)
        engine.describe(self.f["mim"], self.k["x"], self.k["y"], self.k["count"], c.n_orient, c.patch_size,
                        c.grid, c.dominant_ratio, c.rotate_patch, "rift2", capacity=2 * self.K,
                        ws_key="b_describe", out=self.d)
        engine.match(self.d, self.dim, self.rb, self.tb, self.K, ws_key="b_match", out=self.m)

    def run(self):
        self.run_fields()
        self.run_features()

    # number of our kernels one step launches (fields 7 + detect 5 + describe 3 + match 4)
    KERNELS_PER_STEP = 19

    # ---- graphs ------------------------------------------------------------
    def capture(self):
        """Warm up (allocates workspaces and cached tables), then capture.

        Three graphs: the filter bank on each of two image buffers (so a
        host upload can fill one while the other is being read) and the
        detect + describe + match group."""
        self.run()
        torch.cuda.synchronize()
        if self._alt is None:
            self._alt = torch.zeros_like(self.images)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g_a, g_b, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g_a, stream=s):
                self.run_fields()
            self.images, self._alt = self._alt, self.images
            try:
                with torch.cuda.graph(g_b, stream=s):
                    self.run_fields()
            finally:
                self.images, self._alt = self._alt, self.images
            with torch.cuda.graph(g2, stream=s):
                self.run_features()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graphs = (g_a, g2, g_b)
        return self

    def replay_fields(self):
        self.graphs[0].replay()

    def replay_features(self):
        self.graphs[1].replay()

    def step(self):
        if self.graphs is None:
            self.run()
        else:
            self.graphs[0].replay()
            self.graphs[1].replay()

    def run_from_host(self, host_images, steps: int, host_out: dict | None = None):
        """End-to-end steps from host memory: step i uploads host_images[i %
        len] (pinned (B, H, W) float32 tensors) on a copy stream into one of
        two device buffers while the previous step computes, runs the whole
        pipeline on the current stream, and copies the match arrays back into
        `host_out` (pinned tensors shaped like `self.m`).  Enqueues only; the
        caller synchronises."""
        if self.graphs is None:
            self.capture()
        if not isinstance(host_images, (list, tuple)):
            host_images = [host_images]
        cs = torch.cuda.current_stream()
        xs = self._copy_stream = self._copy_stream or torch.cuda.Stream()
        bufs = (self.images, self._alt)
        fields_graph = (self.graphs[0], self.graphs[2])
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        xs.wait_stream(cs)
        with torch.cuda.stream(xs):
            bufs[0].copy_(host_images[0], non_blocking=True)
            ready[0].record(xs)
        for i in range(steps):
            b = i % 2
            if i + 1 < steps:
                with torch.cuda.stream(xs):
                    if i >= 1:
                        xs.wait_event(done[1 - b])           # step i-1 finished reading that buffer
                    bufs[1 - b].copy_(host_images[(i + 1) % len(host_images)], non_blocking=True)
                    ready[1 - b].record(xs)
            cs.wait_event(ready[b])
            fields_graph[b].replay()
            done[b].record(cs)
            self.graphs[1].replay()
            if host_out is not None:
                for k, t in host_out.items():
                    t.copy_(self.m[k], non_blocking=True)
        cs.wait_stream(xs)

    # ---- results -----------------------------------------------------------
    def matches_host(self):
        """Per pair (ref ids, tgt ids, dist) numpy arrays."""
        cnt = self.m["count"].cpu().numpy()
        ref, tgt, dist = (self.m[k].cpu().numpy() for k in ("ref", "tgt", "dist"))
        return [(ref[p, :cnt[p]], tgt[p, :cnt[p]], dist[p, :cnt[p]]) for p in range(self.P)]

    def keypoints_host(self, i: int):
        n = int(self.k["count"][i])
        return {k: self.k[k][i, :n].cpu().numpy() for k in ("x", "y", "response", "kind")}

    def load(self, images: np.ndarray):
        if images.shape != (self.B, self.H, self.W):
            raise ParameterError(f"expected images of shape {(self.B, self.H, self.W)}, got {images.shape}")
        self.images.copy_(torch.from_numpy(np.ascontiguousarray(images, dtype=np.float32)))
