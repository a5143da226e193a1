"""Row-sharded matching of one large pair over G processes.

SURVEY.md 8(e), BASELINE.json configs[3] (one 4096^2 pair, up to 20,000
keypoints per image, the distance matrix row-sharded across GPUs):

1. Every rank runs the filter bank and detection of both images.  They are
   deterministic, so all ranks hold identical keypoint lists.
2. Rank r describes only its contiguous slice [n*r/G, n*(r+1)/G) of each
   image's keypoints (keypoint ids stay global).
3. The descriptor slices are all-gathered.  Image 2's (the targets) are
   needed in full by every rank; image 1's reference rows are needed for
   the float64 distance of each winner.  Concatenating slices in rank order
   reproduces the single-GPU descriptor order exactly.
4. Each rank matches all target descriptors against its own reference slice
   (rift2_match_partial: the tensor-core GEMM with the exact running argmax).
5. The per-target partial bests (16 bytes per target row) are all-gathered
   and combined exactly (rift2_match_finish: variant groups, exact integer
   comparison, ties to the smallest reference keypoint id, float64
   distances, (dist, ref, tgt) order).  The result equals the single-GPU
   match_nn bit for bit.

Collectives: four all-gathers of sizes/rows per image plus one of the
partials; no reduction touches floating point.  The kernels and the
collective are injected (`backend`, `group`), so the same orchestration runs
the GPU path (NCCL) and, in tests/test_multirank.py, a CPU backend under
gloo.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .config import RiftConfig
from .matcher import MatchSet


def kp_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous keypoint slice of `rank` (sizes differ by at most one)."""
    return n * rank // world, n * (rank + 1) // world


def _world(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def gather_rows(t: torch.Tensor, group=None) -> torch.Tensor:
    """Concatenate every rank's rows (dim 0, sizes may differ) in rank order."""
    rank, world = _world(group)
    if world == 1:
        return t
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes)
    pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[:t.shape[0]] = t
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)], dim=0)


def gather_equal(t: torch.Tensor, group=None) -> torch.Tensor:
    """Stack every rank's equally shaped tensor -> (world, *t.shape)."""
    rank, world = _world(group)
    if world == 1:
        return t[None]
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t.contiguous(), group=group)
    return torch.stack(bufs)


class GpuBackend:
    """The CUDA path: every step is one call into the C ABI (engine.*)."""

    DESC_KEYS = ("counts", "sqnorm", "kp", "variant")

    def __init__(self, device=None):
        self.dev = torch.device(device or "cuda")

    def features(self, image, cfg: RiftConfig) -> dict:
        from . import engine
        img = torch.as_tensor(np.asarray(image, dtype=np.float32), device=self.dev)[None]
        f = engine.fields(img, cfg.bank_params())
        k = engine.detect(f["mmin"], f["mmax"], cfg.fast_threshold, cfg.max_keypoints, cfg.patch_size // 2)
        n = int(k["count"][0])
        return {"mim": f["mim"], "x": k["x"][:, :n].contiguous(), "y": k["y"][:, :n].contiguous(), "n": n}

    def describe_slice(self, feat: dict, k0: int, k1: int, cfg: RiftConfig) -> dict:
        from . import engine
        n = k1 - k0
        x = feat["x"][:, k0:k1].contiguous()
        y = feat["y"][:, k0:k1].contiguous()
        if n == 0:
            x = torch.zeros((1, 1), dtype=torch.int32, device=self.dev)
            y = torch.zeros((1, 1), dtype=torch.int32, device=self.dev)
        cnt = torch.tensor([n], dtype=torch.int32, device=self.dev)
        d = engine.describe(feat["mim"], x, y, cnt, cfg.n_orient, cfg.patch_size, cfg.grid, cfg.dominant_ratio,
                            cfg.rotate_patch, "rift2")
        m = int(d["count"][0])
        out = {k: d[k][0, :m].contiguous() for k in self.DESC_KEYS}
        out["kp"] = out["kp"] + k0                           # global keypoint ids
        return out

    @staticmethod
    def _pack(ref: dict, tgt: dict, cap: int):
        dev = ref["counts"].device
        stride = ref["counts"].shape[1] if ref["counts"].dim() == 2 else 224
        desc = {"counts": torch.zeros((2, cap, stride), dtype=torch.float16, device=dev),
                "sqnorm": torch.zeros((2, cap), dtype=torch.int32, device=dev),
                "kp": torch.zeros((2, cap), dtype=torch.int32, device=dev)}
        for b, blk in enumerate((ref, tgt)):
            n = blk["counts"].shape[0]
            desc["counts"][b, :n] = blk["counts"]
            desc["sqnorm"][b, :n] = blk["sqnorm"]
            desc["kp"][b, :n] = blk["kp"]
        desc["count"] = torch.tensor([ref["counts"].shape[0], tgt["counts"].shape[0]], dtype=torch.int32,
                                     device=dev)
        rb = torch.tensor([0], dtype=torch.int32, device=dev)
        tb = torch.tensor([1], dtype=torch.int32, device=dev)
        return desc, rb, tb

    def partial(self, ref_local: dict, tgt_full: dict, dim: int) -> torch.Tensor:
        from . import engine
        n_t = tgt_full["counts"].shape[0]
        cap = max(ref_local["counts"].shape[0], n_t, 1)
        desc, rb, tb = self._pack(ref_local, tgt_full, cap)
        parts = engine.match_partial(desc, dim, rb, tb)
        return parts[0, :n_t].contiguous()

    def finish(self, parts_all: torch.Tensor, ref_full: dict, tgt_full: dict, n_ref_kp: int, n_tgt_kp: int,
               dim: int):
        from . import engine
        G, n_t = parts_all.shape[:2]
        # keypoint ids index per-pair tables of `cap` entries
        cap = max(ref_full["counts"].shape[0], n_t, n_ref_kp, n_tgt_kp, 1)
        desc, rb, tb = self._pack(ref_full, tgt_full, cap)
        parts = torch.zeros((G, 1, cap, 4), dtype=torch.int32, device=parts_all.device)
        parts[:, 0, :n_t] = parts_all
        out = engine.match_finish(parts, desc, dim, rb, tb, n_tgt_kp)
        m = int(out["count"][0])
        return (out["ref"][0, :m].cpu().numpy(), out["tgt"][0, :m].cpu().numpy(),
                out["dist"][0, :m].cpu().numpy())


def match_pair_sharded(ref_image, tgt_image, cfg: RiftConfig | None = None, group=None, backend=None):
    """MatchSet of one pair, matching row-sharded over the ranks of `group`
    (the default process group; a single process works too).  Returns
    (MatchSet, info) with info = per-rank slice sizes and counts."""
    cfg = cfg or RiftConfig()
    backend = backend or GpuBackend()
    rank, world = _world(group)
    dim = cfg.grid * cfg.grid * cfg.n_orient
    feats = [backend.features(img, cfg) for img in (ref_image, tgt_image)]   # replicated
    local, full = [], []
    for f in feats:
        k0, k1 = kp_range(f["n"], rank, world)
        loc = backend.describe_slice(f, k0, k1, cfg)
        local.append(loc)
        full.append({k: gather_rows(v, group) for k, v in loc.items()})
    parts = backend.partial(local[0], full[1], dim)
    parts_all = gather_equal(parts, group)
    ref, tgt, dst = backend.finish(parts_all, full[0], full[1], feats[0]["n"], feats[1]["n"], dim)
    n_r, n_t = full[0]["counts"].shape[0], full[1]["counts"].shape[0]
    pairs = [(int(a), int(b), float(c)) for a, b, c in zip(ref, tgt, dst)]
    info = {"world": world, "rank": rank, "ref_slice": kp_range(feats[0]["n"], rank, world),
            "tgt_slice": kp_range(feats[1]["n"], rank, world), "ref_descriptors": n_r, "tgt_descriptors": n_t}
    return MatchSet(pairs=pairs, mode="rift2", distance_evals=n_r * n_t), info
