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

from .errors import FormatError, ParameterError

MODE_CODES = {"plain": 0, "ring": 1, "rift2": 2}
_MODE_NAMES = {v: k for k, v in MODE_CODES.items()}

# "RIF2" container (ref: descriptor.py:26-32, 255-294): an 11-byte header
# (magic, version u8, n_orient u8, grid u8, count u32 LE) and fixed-size
# records (keypoint id u32, variant u8, mode code u8, float32 LE vector),
# read and written here as one packed numpy record array
_MAGIC, _VERSION = b"RIF2", 1
_HEAD = np.dtype([("magic", "S4"), ("version", "u1"), ("n_orient", "u1"), ("grid", "u1"), ("count", "<u4")])


def _record_dtype(dim: int) -> np.dtype:
    return np.dtype([("kp", "<u4"), ("variant", "u1"), ("mode", "u1"), ("vec", "<f4", (dim,))])


@dataclass(frozen=True)
class Descriptor:
    vector: np.ndarray
    keypoint_id: int
    variant: int
    mode: str
    counts: np.ndarray | None = field(default=None, compare=False, repr=False)
    # the describe call's (n, dim) count matrix and this row in it: lets
    # match_nn gather whole descriptor lists without restacking them
    _src: np.ndarray | None = field(default=None, compare=False, repr=False)
    _row: int = field(default=-1, compare=False, repr=False)


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
    from . import _devcache
    dev = _devcache.lookup(mim.indices)
    if dev is not None:
        return dev
    idx = np.asarray(mim.indices)
    if idx.size and (idx.min() < 1 or idx.max() > mim.n_orient):
        raise ParameterError(f"index map values must lie in [1, {mim.n_orient}]")
    return torch.from_numpy(np.ascontiguousarray(idx.astype(np.uint8))).cuda()


def _kp_arrays(keypoints):
    """int32 coordinates when every keypoint is integral (the detector's
    output), else float64 for rift2_describe_f64 (ref: descriptor.py:105-125
    samples fractional keypoints at floor(x + ux + 0.5))."""
    xs = np.array([k.x for k in keypoints], dtype=np.float64)
    ys = np.array([k.y for k in keypoints], dtype=np.float64)
    if np.any(xs != np.floor(xs)) or np.any(ys != np.floor(ys)):
        return xs, ys
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
    # the reference's vector is counts / ||counts|| (ref: descriptor.py:161-164);
    # the counts are integers, so c.c is exact in any summation order and the
    # row-wise norm and division below are bit-identical to the per-vector ones
    vecs = counts.astype(np.float64)
    vecs /= np.sqrt(np.einsum("ij,ij->i", vecs, vecs))[:, None]
    descs = [Descriptor(vec, k, v, mode, c, counts, i)
             for i, (vec, c, k, v) in enumerate(zip(vecs, counts, kps.tolist(), var.tolist()))]
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


def _write_records(path, n_orient: int, grid: int, kp, variant, mode_code, vec32) -> None:
    dim = grid * grid * n_orient
    rec = np.empty(len(kp), dtype=_record_dtype(dim))
    rec["kp"], rec["variant"], rec["mode"], rec["vec"] = kp, variant, mode_code, vec32
    head = np.array([(_MAGIC, _VERSION, n_orient, grid, len(kp))], dtype=_HEAD)
    with open(path, "wb") as fh:
        fh.write(head.tobytes())
        fh.write(rec.tobytes())


def write_descriptors(path, descriptors, n_orient: int = 6, grid: int = 6) -> None:
    """ref: descriptor.py:255-268 (same bytes)."""
    dim = grid * grid * n_orient
    descriptors = list(descriptors)
    for d in descriptors:
        if np.shape(d.vector) != (dim,):
            raise ParameterError(f"descriptor length {np.shape(d.vector)} does not match {dim}")
    vec = np.array([d.vector for d in descriptors], dtype=np.float64).reshape(len(descriptors), dim)
    _write_records(path, n_orient, grid, [d.keypoint_id for d in descriptors], [d.variant for d in descriptors],
                   [MODE_CODES[d.mode] for d in descriptors], vec.astype("<f4"))


def write_descriptor_counts(path, counts, kp, variant, mode: str = "rift2", n_orient: int = 6,
                            grid: int = 6) -> None:
    """The same container straight from the batched tensors of one image
    (`BatchPipeline.d` / `engine.describe` rows, counts (n, >= dim)): the
    float64 unit vector counts / ||counts|| is formed on the device, rounded
    to float32 as write_descriptors does, and written without building
    Descriptor objects."""
    import torch
    dim = grid * grid * n_orient
    c = counts[:, :dim].to(torch.float64)
    vec = (c / torch.sqrt((c * c).sum(dim=1, keepdim=True))).to(torch.float32).cpu().numpy()
    as_np = (lambda t: t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t))
    _write_records(path, n_orient, grid, as_np(kp), as_np(variant), MODE_CODES[mode], vec)


def read_descriptors(path) -> list:
    """ref: descriptor.py:271-294 (FormatError on a short header, bad magic,
    unknown version or mode code, and truncated records)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _HEAD.itemsize:
        raise FormatError("descriptor file too short for header")
    head = np.frombuffer(raw, dtype=_HEAD, count=1)[0]
    if head["magic"] != _MAGIC:
        raise FormatError(f"bad magic {bytes(head['magic'])!r}")
    if head["version"] != _VERSION:
        raise FormatError(f"unsupported version {int(head['version'])}")
    dim = int(head["grid"]) * int(head["grid"]) * int(head["n_orient"])
    rdt = _record_dtype(dim)
    count = int(head["count"])
    if len(raw) - _HEAD.itemsize < count * rdt.itemsize:
        raise FormatError("descriptor file truncated")
    rec = np.frombuffer(raw, dtype=rdt, count=count, offset=_HEAD.itemsize)
    bad = ~np.isin(rec["mode"], list(_MODE_NAMES))
    if bad.any():
        raise FormatError(f"unknown mode code {int(rec['mode'][bad][0])}")
    vec = rec["vec"].astype(np.float64)
    return [Descriptor(vec[i], int(rec["kp"][i]), int(rec["variant"][i]), _MODE_NAMES[int(rec["mode"][i])])
            for i in range(count)]


def _snap(v: float) -> float:
    """cos / sin snapping of ref: descriptor.py:59-60 (quarter turns exact)."""
    if abs(v) < 1e-12:
        return 0.0
    if abs(abs(v) - 1.0) < 1e-12:
        return float(np.copysign(1.0, v))
    return float(v)


def extract_patch(mim, keypoint, size: int, angle: float = 0.0, with_amplitude: bool = True):
    """ref: descriptor.py:85-125 -- size x size index patch on a grid rotated
    by `angle` about the keypoint, None when any sample leaves the map.  The
    axis-aligned crop is a view (as the reference returns); rotated grids are
    gathered by rift2_extract_patch with the reference's float64 offsets and
    rounding."""
    import torch
    from . import engine
    from .mim import IndexMap
    h, w = mim.shape
    if angle == 0.0:
        x0 = int(np.floor(keypoint.x + 1.0 - size / 2.0))
        y0 = int(np.floor(keypoint.y + 1.0 - size / 2.0))
        if x0 < 0 or y0 < 0 or x0 + size > w or y0 + size > h:
            return None
        return mim.region(y0, y0 + size, x0, x0 + size)
    idx = torch.from_numpy(np.ascontiguousarray(mim.indices, dtype=np.int32)).cuda()
    amp = torch.from_numpy(np.ascontiguousarray(mim.max_amplitude, dtype=np.float64)).cuda() if with_amplitude else None
    c, s = _snap(np.cos(angle)), _snap(np.sin(angle))
    oi, oa, oob = engine.extract_patch(idx, amp, float(keypoint.x), float(keypoint.y), int(size), c, s, with_amplitude)
    if oob:
        return None
    amplitude = oa.cpu().numpy() if with_amplitude else np.broadcast_to(0.0, (size, size))
    return IndexMap(oi.cpu().numpy().astype(np.asarray(mim.indices).dtype, copy=False), amplitude, mim.n_orient)


def encode(patch, grid: int = 6, weighted: bool = False):
    """ref: descriptor.py:145-164 -- concatenated per-cell index histograms,
    L2-normalised; None for the all-zero vector (weighted mode only).  The
    cell counts come from rift2_patch_counts; the float64 normalisation is the
    reference's own (v / ||v||), as describe_* rebuilds its vectors."""
    import torch
    from . import engine
    from .mim import _check_values
    idx = np.asarray(patch.indices)
    h, w = idx.shape
    if h != w or h % grid != 0:
        raise ParameterError(f"patch {h}x{w} does not divide into {grid}x{grid} cells")
    _check_values(idx, patch.n_orient)
    d_idx = torch.from_numpy(np.ascontiguousarray(idx[None], dtype=np.int32)).cuda()
    amp = torch.from_numpy(np.ascontiguousarray(np.asarray(patch.max_amplitude, dtype=np.float64)[None])).cuda() \
        if weighted else None
    _, cells = engine.patch_counts(d_idx, amp, patch.n_orient, grid, hist=False, cells=True)
    vector = cells[0].cpu().numpy()
    norm = np.linalg.norm(vector)
    if norm == 0:
        return None
    return vector / norm
