"""Row-sharded matching of one large pair over G processes.

SURVEY.md 8(e), BASELINE.json configs[3] (one 4096^2 pair, up to 20,000
keypoints per image, the distance matrix row-sharded across GPUs):

1. Every rank runs the filter bank and detection of both images.  They are
   deterministic, so all ranks hold identical keypoint lists.
2. Rank r describes only its contiguous slice [n*r/G, n*(r+1)/G) of each
   image's keypoints (keypoint ids stay global).
3. Image 2's descriptor slices (the targets) are all-gathered -- the one
   data-path collective `north_star` names.  Concatenating slices in rank
   order reproduces the single-GPU descriptor order exactly.  Image 1's
   reference rows never leave their rank.
4. Each rank matches all target descriptors against its own reference slice
   (rift2_match_partial: the tensor-core GEMM with the exact running argmax).
5. The per-target partial bests (16 bytes per target row) are all-gathered
   and combined exactly on every rank (rift2_match_finish on the local
   reference slice: variant groups, exact integer comparison, ties to the
   smallest reference keypoint id).  The winner of each target keypoint is
   the same on every rank; its float64 distance is computed by the rank
   that owns the winner's reference rows (+inf elsewhere).
6. The (ref, tgt, dist) triples (16 bytes per target keypoint) are
   all-gathered, each target keeps the finite distance, and the set is
   sorted by (dist, ref, tgt).  The result equals the single-GPU match_nn
   bit for bit.

Collectives: all-gathers of image 2's descriptor rows, of the partials and
of the per-target triples; no reduction touches floating point.  The kernels
and the collective are injected (`backend`, `group`), so the same
orchestration runs the GPU path (NCCL) and, in tests/test_multirank.py, a
CPU backend under gloo.
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

    def finish_local(self, parts_all: torch.Tensor, ref_local: dict, tgt_full: dict, n_ref_kp: int,
                     n_tgt_kp: int, dim: int):
        """Exact combine of the gathered partials against this rank's
        reference slice -> (ref, tgt, dist) numpy arrays, one per target
        keypoint; dist is +inf where the winner's rows live on another rank."""
        from . import engine
        G, n_t = parts_all.shape[:2]
        n_r = ref_local["counts"].shape[0]
        if n_r == 0 or n_t == 0:
            return np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, np.float64)
        # keypoint ids index per-pair tables of `cap` entries
        cap = max(n_r, n_t, n_ref_kp, n_tgt_kp, 1)
        desc, rb, tb = self._pack(ref_local, tgt_full, cap)
        parts = torch.zeros((G, 1, cap, 4), dtype=torch.int32, device=parts_all.device)
        parts[:, 0, :n_t] = parts_all
        out = engine.match_finish(parts, desc, dim, rb, tb, n_tgt_kp)
        m = int(out["count"][0])
        return (out["ref"][0, :m].cpu().numpy(), out["tgt"][0, :m].cpu().numpy(),
                out["dist"][0, :m].cpu().numpy())


def merge_triples(parts) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Every rank's (ref, tgt, dist) triples -> one per target keypoint with
    the finite distance (supplied by the winner's owner), sorted by (dist,
    ref, tgt) like ref: matcher.py:143-146."""
    ref = np.concatenate([np.asarray(p[0], np.int64) for p in parts]) if parts else np.zeros(0, np.int64)
    tgt = np.concatenate([np.asarray(p[1], np.int64) for p in parts]) if parts else np.zeros(0, np.int64)
    dst = np.concatenate([np.asarray(p[2], np.float64) for p in parts]) if parts else np.zeros(0)
    best = {}
    for r, t, d in zip(ref.tolist(), tgt.tolist(), dst.tolist()):
        cur = best.get(t)
        if cur is not None and cur[0] != r:
            raise RuntimeError(f"ranks disagree on the winner of target keypoint {t}: {cur[0]} vs {r}")
        if cur is None or d < cur[1]:
            best[t] = (r, d)
    trip = sorted(((r, t, d) for t, (r, d) in best.items()), key=lambda p: (p[2], p[0], p[1]))
    if any(not np.isfinite(d) for _, _, d in trip):
        raise RuntimeError("a winner's distance was supplied by no rank")
    return (np.array([p[0] for p in trip], np.int64), np.array([p[1] for p in trip], np.int64),
            np.array([p[2] for p in trip], np.float64))


def gather_triples(ref, tgt, dst, group=None):
    """All-gather each rank's triples (sizes may differ) as a list per rank."""
    rank, world = _world(group)
    if world == 1:
        return [(ref, tgt, dst)]
    packed = torch.from_numpy(np.stack([np.asarray(ref, np.float64), np.asarray(tgt, np.float64),
                                        np.asarray(dst, np.float64)], 1)) if len(ref) else torch.zeros((0, 3),
                                                                                                       dtype=torch.float64)
    dev = torch.device("cuda", torch.cuda.current_device()) if (dist.get_backend(group) == "nccl") else torch.device("cpu")
    n = torch.tensor([packed.shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(x.item()) for x in sizes]
    m = max(max(sizes), 1)
    pad = torch.zeros((m, 3), dtype=torch.float64, device=dev)
    pad[:packed.shape[0]] = packed.to(dev)
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    out = []
    for b, k in zip(bufs, sizes):
        a = b[:k].cpu().numpy()
        out.append((a[:, 0].astype(np.int64), a[:, 1].astype(np.int64), a[:, 2]))
    return out


def match_pair_sharded(ref_image, tgt_image, cfg: RiftConfig | None = None, group=None, backend=None):
    """MatchSet of one pair, matching row-sharded over the ranks of `group`
    (the default process group; a single process works too).  Returns
    (MatchSet, info) with info = per-rank slice sizes and counts."""
    cfg = cfg or RiftConfig()
    backend = backend or GpuBackend()
    rank, world = _world(group)
    dim = cfg.grid * cfg.grid * cfg.n_orient
    feats = [backend.features(img, cfg) for img in (ref_image, tgt_image)]   # replicated
    slices = [kp_range(f["n"], rank, world) for f in feats]
    ref_local = backend.describe_slice(feats[0], *slices[0], cfg)
    tgt_local = backend.describe_slice(feats[1], *slices[1], cfg)
    tgt_full = {k: gather_rows(v, group) for k, v in tgt_local.items()}     # image 2 only
    parts = backend.partial(ref_local, tgt_full, dim)
    parts_all = gather_equal(parts, group)
    mine = backend.finish_local(parts_all, ref_local, tgt_full, feats[0]["n"], feats[1]["n"], dim)
    ref, tgt, dst = merge_triples(gather_triples(*mine, group=group))
    n_r_local = int(ref_local["counts"].shape[0])
    n_r = int(sum(int(x) for x in gather_equal(torch.tensor([n_r_local], device=parts.device), group).view(-1)))
    n_t = tgt_full["counts"].shape[0]
    pairs = [(int(a), int(b), float(c)) for a, b, c in zip(ref, tgt, dst)]
    info = {"world": world, "rank": rank, "ref_slice": slices[0], "tgt_slice": slices[1],
            "ref_descriptors": n_r, "ref_descriptors_local": n_r_local, "tgt_descriptors": n_t}
    return MatchSet(pairs=pairs, mode="rift2", distance_evals=n_r * n_t), info
