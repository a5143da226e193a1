"""Batched tensor API: the throughput path used by bench.py.

A BatchPipeline owns every device buffer for `n_pairs` image pairs of one
size (images interleaved [ref0, tgt0, ref1, tgt1, ...]) and runs the four
stages back to back on the current stream with no host synchronisation.
The two stage groups (filter bank; detect + describe + match) are captured
into CUDA graphs after a warm-up, so a step is two graph launches.

Throughput mode (`capture_pipelined` / `pipelined_step` /
`run_from_host_pipelined`): the filter bank of batch i runs on one stream
while detect / describe / match of batch i-1 runs on another, on
double-buffered field maps -- each step still completes one batch, one step
later, with results identical to `step()`.
"""

from __future__ import annotations

import itertools

import numpy as np
import torch

from . import engine
from .config import RiftConfig
from .errors import ParameterError


_INSTANCE_IDS = itertools.count()


class BatchPipeline:
    def __init__(self, n_pairs: int, height: int, width: int, cfg: RiftConfig | None = None, device=None):
        self.cfg = cfg or RiftConfig()
        # descriptor mode and rows per keypoint (ref: pipeline.py:53-64): rift2
        # one or two per keypoint on both sides; ring n_orient cyclic layers on
        # the reference side against plain targets; plain one per keypoint
        modes = {"rift2": ("rift2", 2), "ring": ("ring_pipeline", self.cfg.n_orient), "plain": ("plain", 1)}
        if self.cfg.mode not in modes:
            raise ParameterError(f"unknown mode {self.cfg.mode!r}")
        self.desc_mode, per = modes[self.cfg.mode]
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
                      mim=torch.empty((B, H, W), dtype=torch.uint8, device=d),
                      range=torch.zeros((B, 2, 2), dtype=torch.int64, device=d))
        self.k = dict(x=torch.zeros((B, K), dtype=torch.int32, device=d),
                      y=torch.zeros((B, K), dtype=torch.int32, device=d),
                      response=torch.zeros((B, K), dtype=torch.float64, device=d),
                      kind=torch.zeros((B, K), dtype=torch.uint8, device=d),
                      count=torch.zeros((B,), dtype=torch.int32, device=d))
        cap = per * K
        self.cap = cap
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
        # workspace keys private to this pipeline: its captured graphs hold
        # the scratch addresses, so no other caller may grow or share them
        self._ws = f"bp{next(_INSTANCE_IDS)}_"
        self.graphs = None
        self._alt = None
        self._copy_stream = None

    # ---- stages (eager) --------------------------------------------------
    def run_fields(self, images=None, f=None, ws: str = "b_"):
        ws = self._ws + ws
        engine.fields(self.images if images is None else images, self.bank, out=self.f if f is None else f,
                      ws_key=ws + "fields")

    def run_features(self, f=None, ws: str = "b_"):
        ws = self._ws + ws
        f = self.f if f is None else f
        c = self.cfg
        engine.detect(f["mmin"], f["mmax"], c.fast_threshold, self.K, c.patch_size // 2, ws_key=ws + "detect",
                      out=self.k, moment_range=f["range"])
        engine.describe(f["mim"], self.k["x"], self.k["y"], self.k["count"], c.n_orient, c.patch_size, c.grid,
                        c.dominant_ratio, c.rotate_patch, self.desc_mode, capacity=self.cap, ws_key=ws + "describe",
                        out=self.d)
        engine.match(self.d, self.dim, self.rb, self.tb, self.K, ws_key=ws + "match", out=self.m)

    def run(self):
        self.run_fields()
        self.run_features()

    # our kernels per step: fields 10 (with the moment-range init) + detect 9
    # (no k_minmax: the PC pass reduced the maps) + describe 3 (the shift-byte
    # copy of the index maps, the dense cell sums, the per-keypoint kernel) +
    # match 7
    KERNELS_PER_STEP = 29

    # ---- graphs ------------------------------------------------------------
    def capture(self):
        """Warm up (allocates workspaces and cached tables), then capture the
        filter bank on each of two image buffers (a host upload can fill one
        while the other is read) and the detect + describe + match group."""
        self.run()
        torch.cuda.synchronize()
        if self._alt is None:
            self._alt = torch.zeros_like(self.images)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g_a, g_b, g_d = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g_a, stream=s):
                self.run_fields()
            with torch.cuda.graph(g_b, stream=s):
                self.run_fields(images=self._alt)
            with torch.cuda.graph(g_d, stream=s):
                self.run_features()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graphs = {"fields": (g_a, g_b), "features": g_d}
        return self

    def replay_fields(self, buf: int = 0):
        self.graphs["fields"][buf].replay()

    def replay_features(self):
        self.graphs["features"].replay()

    def step(self):
        if self.graphs is None:
            self.run()
        else:
            self.replay_fields()
            self.replay_features()

    def run_from_host(self, host_images, steps: int, host_out: dict | None = None):
        """End-to-end steps from host memory: step i uploads host_images[i %
        len] (pinned (B, H, W) float32 tensors) on a copy stream into one of
        two device buffers while the previous step computes, runs the whole
        pipeline on the current stream, and copies results back into
        `host_out` (pinned tensors keyed like `_result`: match arrays and the
        keypoint coordinates they index).  Enqueues only; the caller
        synchronises."""
        if self.graphs is None:
            self.capture()
        if not isinstance(host_images, (list, tuple)):
            host_images = [host_images]
        cs = torch.cuda.current_stream()
        xs = self._copy_stream = self._copy_stream or torch.cuda.Stream()
        bufs = (self.images, self._alt)
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
            self.replay_fields(b)
            done[b].record(cs)
            self.replay_features()
            if host_out is not None:
                for k, t in host_out.items():
                    t.copy_(self._result(k), non_blocking=True)
        cs.wait_stream(xs)

    # ---- cross-step pipeline --------------------------------------------------
    # Step i runs the filter bank of batch i (stream 1) concurrently with
    # detect / describe / match of batch i-1 (stream 2), on double-buffered
    # field maps; every pair still goes through the whole path, one step
    # later.  After pipelined_step(p) the match arrays hold the batch whose
    # filter bank ran in the previous pipelined step.
    def capture_pipelined(self):
        if self.graphs is None:
            self.capture()
        if getattr(self, "_f2", None) is None:
            self._f2 = {k: torch.zeros_like(v) for k, v in self.f.items()}
        fbuf = (self.f, self._f2)
        imgs = (self.images, self._alt)
        for p in (0, 1):                                   # warm-up: allocate workspaces
            self.run_fields(imgs[p], fbuf[p], "p_")
            self.run_features(fbuf[1 - p], "p_")
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        side = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        graphs, feats = [], []
        with torch.cuda.stream(s):
            for p in (0, 1):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    side.wait_stream(s)
                    with torch.cuda.stream(side):
                        self.run_features(fbuf[1 - p], "p_")
                    self.run_fields(imgs[p], fbuf[p], "p_")
                    s.wait_stream(side)
                graphs.append(g)
            # drain steps: the features of the last batch alone, on either buffer
            for p in (0, 1):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    self.run_features(fbuf[p], "p_")
                feats.append(g)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graphs["pipe"] = tuple(graphs)
        self.graphs["pipe_features"] = tuple(feats)
        return self

    def pipelined_step(self, parity: int):
        self.graphs["pipe"][parity & 1].replay()

    def run_from_host_pipelined(self, host_images, steps: int, host_out: dict | None = None):
        """As run_from_host, pipelined: step i uploads batch i+1 on the copy
        stream, runs the filter bank of batch i next to the features of batch
        i-1, and copies batch i-1's match arrays back.  The first step is the
        filter bank of batch 0 alone and the last the features of batch
        steps-1 alone, so `steps` batches are processed with no other work.
        Enqueues only."""
        if "pipe" not in (self.graphs or {}):
            self.capture_pipelined()
        if not isinstance(host_images, (list, tuple)):
            host_images = [host_images]
        cs = torch.cuda.current_stream()
        xs = self._copy_stream = self._copy_stream or torch.cuda.Stream()
        bufs = (self.images, self._alt)
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        xs.wait_stream(cs)
        with torch.cuda.stream(xs):
            bufs[0].copy_(host_images[0], non_blocking=True)
            ready[0].record(xs)
        for i in range(steps + 1):
            b = i % 2
            if i + 1 < steps:
                with torch.cuda.stream(xs):
                    if i >= 1:
                        xs.wait_event(done[1 - b])
                    bufs[1 - b].copy_(host_images[(i + 1) % len(host_images)], non_blocking=True)
                    ready[1 - b].record(xs)
            if i < steps:
                cs.wait_event(ready[b])
            if i == 0:
                self.graphs["fields"][0].replay()          # fields(images -> f): the fields half of pipe[0]
            elif i == steps:
                self.graphs["pipe_features"][1 - b].replay()
            else:
                self.pipelined_step(b)
            done[b].record(cs)
            if i >= 1 and host_out is not None:            # batch i-1 is complete
                for k, t in host_out.items():
                    t.copy_(self._result(k), non_blocking=True)
        cs.wait_stream(xs)

    # ---- results -----------------------------------------------------------
    def _result(self, key: str) -> torch.Tensor:
        """A result array by name: match arrays (ref, tgt, dist, count) or the
        keypoints they index (kp_x, kp_y, kp_count: (2 * n_pairs, K), the
        reference image of pair p at row 2p, its target at 2p + 1)."""
        if key.startswith("kp_"):
            return self.k[key[3:]]
        return self.m[key]

    def result_shapes(self, keys) -> dict:
        return {k: (tuple(self._result(k).shape), self._result(k).dtype) for k in keys}

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
