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
    # The batch is processed as (up to) two halves of pairs with their own
    # workspaces.  In the captured step the second half's filter bank runs
    # while the first half's detect / describe / match (whose per-image
    # kernels leave most SMs idle) runs on a second stream.
    def _halves(self):
        if self.P < 2:
            return [(0, self.P)]
        h = self.P // 2
        return [(0, h), (h, self.P)]

    def run_fields_half(self, i: int, images=None):
        p0, p1 = self._halves()[i]
        img = self.images if images is None else images
        f = {k: v[2 * p0:2 * p1] for k, v in self.f.items()}
        engine.fields(img[2 * p0:2 * p1], self.bank, out=f, ws_key=f"b_fields{i}")

    def run_features_half(self, i: int):
        p0, p1 = self._halves()[i]
        c = self.cfg
        sl = slice(2 * p0, 2 * p1)
        k = {n: v[sl] for n, v in self.k.items()}
        d = {n: v[sl] for n, v in self.d.items()}
        m = {n: v[p0:p1] for n, v in self.m.items()}
        n = p1 - p0
        engine.detect(self.f["mmin"][sl], self.f["mmax"][sl], c.fast_threshold, self.K, c.patch_size // 2,
                      ws_key=f"b_detect{i}", out=k)
        engine.describe(self.f["mim"][sl], k["x"], k["y"], k["count"], c.n_orient, c.patch_size,
                        c.grid, c.dominant_ratio, c.rotate_patch, "rift2", capacity=2 * self.K,
                        ws_key=f"b_describe{i}", out=d)
        engine.match(d, self.dim, self.rb[:n], self.tb[:n], self.K, ws_key=f"b_match{i}", out=m)

    def run_fields(self, images=None):
        for i in range(len(self._halves())):
            self.run_fields_half(i, images)

    def run_features(self):
        for i in range(len(self._halves())):
            self.run_features_half(i)

    def run(self):
        self.run_fields()
        self.run_features()

    def _run_overlapped(self, images, side: torch.cuda.Stream):
        """Enqueue one step: F0, then F1 on this stream while D0 runs on `side`, then D1."""
        main = torch.cuda.current_stream()
        nh = len(self._halves())
        self.run_fields_half(0, images)
        if nh == 1:
            self.run_features_half(0)
            return
        side.wait_stream(main)
        with torch.cuda.stream(side):
            self.run_features_half(0)
        self.run_fields_half(1, images)
        self.run_features_half(1)
        main.wait_stream(side)

    @property
    def KERNELS_PER_STEP(self):
        # our kernels per step: per half, fields 7 + detect 5 + describe 3 + match 4
        return 19 * len(self._halves())

    # ---- graphs ------------------------------------------------------------
    def capture(self):
        """Warm up (allocates workspaces and cached tables), then capture.

        Graphs: the overlapped whole step on each of two image buffers (a
        host upload can fill one while the other is being read), plus the
        filter bank alone (both halves, one stream) and the feature stages
        alone, used by bench.py to time the filter bank by itself."""
        self.run()
        torch.cuda.synchronize()
        if self._alt is None:
            self._alt = torch.zeros_like(self.images)
        s = torch.cuda.Stream()
        side = self._side = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g_a, g_b = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        g_f, g_d = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g_a, stream=s):
                self._run_overlapped(self.images, side)
            with torch.cuda.graph(g_b, stream=s):
                self._run_overlapped(self._alt, side)
            with torch.cuda.graph(g_f, stream=s):
                self.run_fields()
            with torch.cuda.graph(g_d, stream=s):
                self.run_features()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graphs = {"step": (g_a, g_b), "fields": g_f, "features": g_d}
        return self

    def replay_fields(self):
        self.graphs["fields"].replay()

    def replay_features(self):
        self.graphs["features"].replay()

    def step(self):
        if self.graphs is None:
            self.run()
        else:
            self.graphs["step"][0].replay()

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
        step_graph = self.graphs["step"]
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
            step_graph[b].replay()
            done[b].record(cs)
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
