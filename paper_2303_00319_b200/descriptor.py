"""Dominant-index descriptors, drop-in for ref: pkg/src/rift2/descriptor.py:35-254.

describe_rift2 / describe_ring / describe_plain run the CUDA descriptor
kernels (csrc/describe.cu).  The kernels emit exact integer cell-histogram
counts; the float64 unit vector of each Descriptor is rebuilt here with the
reference's own operations (counts / ||counts||, ref: descriptor.py:161-164),
so vectors are bit-identical to the reference's.  The counts ride along on
the Descriptor (field `counts`) so match_nn can use the exact tensor-core
path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ParameterError

MODE_CODES = {"plain": 0, "ring": 1, "rift2": 2}


@dataclass(frozen=True)
class Descriptor:
    vector: np.ndarray
    keypoint_id: int
    variant: int
    mode: str
    counts: np.ndarray | None = field(default=None, compare=False, repr=False)


@dataclass
class DescriptorSet:
    descriptors: list
    skipped: int

    def __len__(self):
        return len(self.descriptors)

    def __iter__(self):
        return iter(self.descriptors)


def _mim_device(mim):
    import torch
    dev = getattr(mim, "device", None)
    if dev is not None:
        return dev
    idx = np.asarray(mim.indices)
    if idx.size and (idx.min() < 1 or idx.max() > mim.n_orient):
        raise ParameterError(f"index map values must lie in [1, {mim.n_orient}]")
    return torch.from_numpy(np.ascontiguousarray(idx.astype(np.uint8))).cuda()


def _kp_arrays(keypoints):
    xs = np.array([k.x for k in keypoints], dtype=np.float64)
    ys = np.array([k.y for k in keypoints], dtype=np.float64)
    if np.any(xs != np.floor(xs)) or np.any(ys != np.floor(ys)):
        raise ParameterError("keypoints must have integer coordinates (detector output always does)")
    return xs.astype(np.int32), ys.astype(np.int32)


def _run(mim, keypoints, patch_size, grid, ratio, rotate, weighted, mode) -> DescriptorSet:
    import torch
    from . import engine
    if weighted:
        raise ParameterError("amplitude-weighted histograms are not supported by the GPU descriptor")
    if patch_size % grid != 0:
        raise ParameterError(f"patch {patch_size}x{patch_size} does not divide into {grid}x{grid} cells")
    if not keypoints:
        return DescriptorSet([], 0)
    xs, ys = _kp_arrays(keypoints)
    m = _mim_device(mim)
    x = torch.from_numpy(xs).cuda()[None]
    y = torch.from_numpy(ys).cuda()[None]
    cnt = torch.tensor([len(xs)], dtype=torch.int32, device="cuda")
    out = engine.describe(m[None], x, y, cnt, int(mim.n_orient), int(patch_size), int(grid), float(ratio),
                          bool(rotate), mode)
    n = int(out["count"][0])
    dim = grid * grid * int(mim.n_orient)
    counts = out["counts"][0, :n, :dim].to(torch.int64).cpu().numpy()
    kps = out["kp"][0, :n].cpu().numpy()
    var = out["variant"][0, :n].cpu().numpy()
    descs = []
    for c, k, v in zip(counts, kps, var):
        vec = c.astype(np.float64)
        descs.append(Descriptor(vec / np.linalg.norm(vec), int(k), int(v), mode, c))
    return DescriptorSet(descs, int(out["skipped"][0]))


def describe_rift2(mim, keypoints, patch_size: int = 96, grid: int = 6, dominant_ratio: float = 0.8,
                   rotate_patch: bool = True, weighted: bool = False) -> DescriptorSet:
    """ref: descriptor.py:179-216."""
    if not 0 < dominant_ratio <= 1:
        raise ParameterError("dominant_ratio must be in (0, 1]")
    return _run(mim, keypoints, patch_size, grid, dominant_ratio, rotate_patch, weighted, "rift2")


def describe_ring(mim, keypoints, patch_size: int = 96, grid: int = 6, weighted: bool = False) -> DescriptorSet:
    """ref: descriptor.py:219-236."""
    return _run(mim, keypoints, patch_size, grid, 0.8, False, weighted, "ring")


def describe_plain(mim, keypoints, patch_size: int = 96, grid: int = 6, weighted: bool = False) -> DescriptorSet:
    """ref: descriptor.py:239-254."""
    return _run(mim, keypoints, patch_size, grid, 0.8, False, weighted, "plain")
