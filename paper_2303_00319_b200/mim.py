"""Maximum index map and its ring algebra, drop-in for ref: pkg/src/rift2/mim.py.
On the pipeline path the map is produced by the fused filter-bank kernel
(csrc/fields.cu) and consumed by the fused descriptor kernel
(csrc/describe.cu); the reference's step-by-step functions run on their own
kernels (rift2_build_mim, rift2_patch_counts, rift2_remap_indices)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ParameterError


@dataclass(frozen=True)
class IndexMap:
    indices: np.ndarray        # int32 in [1, n_orient]
    max_amplitude: np.ndarray  # float64
    n_orient: int

    def __post_init__(self):
        if np.shape(self.indices) != np.shape(self.max_amplitude):
            raise ParameterError("indices and max_amplitude shapes differ")

    @property
    def shape(self):
        return self.indices.shape

    def region(self, y0: int, y1: int, x0: int, x1: int) -> "IndexMap":
        return IndexMap(self.indices[y0:y1, x0:x1], self.max_amplitude[y0:y1, x0:x1], self.n_orient)


def _dev_int32(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def build_mim(a_o) -> IndexMap:
    """ref: mim.py:43-55 -- first argmax over the channel axis, 1-based
    (rift2_build_mim, float64 comparisons: ties resolve as the reference's)."""
    import torch
    from . import engine
    channels = np.asarray(a_o)
    if channels.ndim != 3 or channels.shape[0] < 2:
        raise ParameterError(f"need >= 2 stacked channels of equal size, got shape {channels.shape}")
    idx, amax = engine.build_mim(torch.from_numpy(np.ascontiguousarray(channels, dtype=np.float64)).cuda())
    return IndexMap(indices=idx.cpu().numpy(), max_amplitude=amax.cpu().numpy(), n_orient=channels.shape[0])


def _check_values(indices, n: int) -> None:
    # 0 is never counted (the reference drops bin 0); values above n have no bin
    if indices.size and (indices.min() < 0 or indices.max() > n):
        raise ParameterError(f"index values must lie in [0, {n}]")


def patch_histogram(patch: IndexMap, weighted: bool = False) -> np.ndarray:
    """ref: mim.py:58-66 -- counts (or amplitude mass) per index value
    (rift2_patch_counts)."""
    import torch
    from . import engine
    idx = np.asarray(patch.indices)
    if idx.size == 0:
        raise ParameterError("empty patch")
    _check_values(idx, patch.n_orient)
    flat = idx.reshape(1, 1, -1)
    amp = torch.from_numpy(np.ascontiguousarray(np.asarray(patch.max_amplitude, dtype=np.float64).reshape(1, 1, -1))).cuda() \
        if weighted else None            # one 1 x size "patch": the histogram ignores the shape
    h, _ = engine.patch_counts(_dev_int32(flat), amp, patch.n_orient)
    counts = h[0].cpu().numpy()
    return counts if weighted else counts.astype(np.int64)


def dominant_indices(histogram, ratio: float = 0.8) -> list:
    """ref: mim.py:69-91 -- the peak bin, plus the runner-up when it reaches
    `ratio` of the peak (inclusive); runner-up ties go to the bin cyclically
    closest after the peak.  A selection over n_orient numbers: the batched
    descriptor kernel applies the same rule per keypoint on the device."""
    hist = np.asarray(histogram, dtype=np.float64)
    if hist.sum() <= 0:
        raise ParameterError("histogram has no mass")
    n = len(hist)
    peak = int(np.argmax(hist))
    others = np.delete(np.arange(n), peak)
    result = [peak + 1]
    if len(others):
        runner = hist[others].max()
        if runner >= ratio * hist[peak]:
            tied = others[hist[others] == runner]
            result.append(int(tied[np.argmin((tied - peak) % n)]) + 1)
    return result


def _remapped(patch: IndexMap, pivot: int, kind: int) -> IndexMap:
    from . import engine
    n = patch.n_orient
    if not 1 <= pivot <= n:
        raise ParameterError(f"{'dominant index' if kind == 0 else 'initial layer'} {pivot} outside [1, {n}]")
    idx = np.asarray(patch.indices)
    d = _dev_int32(idx)
    engine.remap_indices(d, n, int(pivot), kind)
    return IndexMap(d.cpu().numpy().astype(idx.dtype, copy=False), patch.max_amplitude, n)


def recode(patch: IndexMap, dominant: int) -> IndexMap:
    """ref: mim.py:117-125 -- renumber so `dominant` becomes 1, ring order kept
    (rift2_remap_indices kind 0)."""
    return _remapped(patch, dominant, 0)


def cyclic_shift(patch: IndexMap, initial_layer: int) -> IndexMap:
    """ref: mim.py:128-136 -- re-base the channel ring on `initial_layer`
    (rift2_remap_indices kind 1)."""
    return _remapped(patch, initial_layer, 1)


def save_index_map_pgm(mim: IndexMap, path) -> None:
    """ref: mim.py:139-144 -- 8-bit PGM dump (values x42) for inspection."""
    data = (np.asarray(mim.indices).astype(np.uint16) * 42).clip(0, 255).astype(np.uint8)
    header = f"P5\n{data.shape[1]} {data.shape[0]}\n255\n".encode("ascii")
    with open(path, "wb") as fh:
        fh.write(header + data.tobytes())
