"""FAST keypoints, drop-in for ref: pkg/src/rift2/detector.py:29-163.

detect_fast / detect_keypoints run the CUDA detector (csrc/detect.cu)
through the C ABI.  When the PCField came from this package's
compute_fields, the GPU's float32 maps are used directly (the float64
arrays in the PCField hold exactly those values); otherwise the caller's
float64 maps are uploaded and scored in float64.  Either way the result is
bit-identical to the reference's detector run on the same map values.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _devcache
from .errors import ParameterError

ARC_LENGTH = 9
_CIRCLE = np.array([(0, -3), (1, -3), (2, -2), (3, -1), (3, 0), (3, 1), (2, 2), (1, 3),
                    (0, 3), (-1, 3), (-2, 2), (-3, 1), (-3, 0), (-3, -1), (-2, -2), (-1, -3)])
_KINDS = ("corner", "edge")


@dataclass(frozen=True)
class Keypoint:
    x: float
    y: float
    response: float
    kind: str

    def to_json_dict(self) -> dict:
        return {"x": self.x, "y": self.y, "response": self.response, "kind": self.kind}

    @classmethod
    def from_json_dict(cls, d: dict) -> "Keypoint":
        return cls(x=float(d["x"]), y=float(d["y"]), response=float(d["response"]), kind=str(d["kind"]))


def keypoints_xy(keypoints) -> np.ndarray:
    return np.array([(k.x, k.y) for k in keypoints], dtype=np.float64).reshape(-1, 2)


def keypoints_to_json(keypoints) -> list:
    return [k.to_json_dict() for k in keypoints]


def keypoints_from_json(items) -> list:
    return [Keypoint.from_json_dict(d) for d in items]


def _to_list(out, b: int, kind_names=_KINDS) -> list:
    n = int(out["count"][b])
    xs = out["x"][b, :n].cpu().numpy()
    ys = out["y"][b, :n].cpu().numpy()
    rs = out["response"][b, :n].cpu().numpy()
    ks = out["kind"][b, :n].cpu().numpy()
    return [Keypoint(x=float(x), y=float(y), response=float(r), kind=kind_names[int(k)])
            for x, y, r, k in zip(xs, ys, rs, ks)]


def _device_map(arr):
    import torch
    if isinstance(arr, torch.Tensor):
        t = arr.detach()
        if not t.is_cuda:
            t = t.cuda()
        if t.dtype not in (torch.float32, torch.float64):
            t = t.double()
        if not bool(torch.isfinite(t).all()):
            raise ParameterError("score map contains non-finite values")
        return t
    a = np.asarray(arr, dtype=np.float64)
    if a.ndim != 2:
        raise ParameterError(f"expected a 2-D map, got shape {a.shape}")
    if not np.all(np.isfinite(a)):
        raise ParameterError("score map contains non-finite values")
    if not a.flags.writeable:             # read-only maps of compute_fields: torch wants a writable source
        a = a.copy()
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def detect_fast(score_map, threshold: float, max_points: int, border_margin: int = 0,
                kind: str = "corner") -> list:
    """ref: detector.py:87-113."""
    from . import engine
    if threshold <= 0:
        raise ParameterError("FAST threshold must be positive")
    m = _device_map(score_map)
    out = engine.detect(m[None], None, float(threshold), int(max_points), int(border_margin), single_map=True)
    return _to_list(out, 0, (kind, kind))


def detect_keypoints(pc, threshold: float = 0.001, max_points: int = 5000, patch_size: int = 96) -> list:
    """ref: detector.py:140-155 -- corners of moment_min and edges of
    moment_max, 2-px greedy merge, capped."""
    from . import engine
    h, w = pc.shape
    if h < patch_size or w < patch_size:
        raise ParameterError(f"image {h}x{w} smaller than the {patch_size}-pixel descriptor patch")
    if threshold <= 0:
        raise ParameterError("FAST threshold must be positive")
    dmin, dmax = _devcache.lookup(pc.moment_min), _devcache.lookup(pc.moment_max)
    if dmin is not None and dmax is not None:
        mins, maxs = dmin[None], dmax[None]
    else:
        mins, maxs = _device_map(pc.moment_min)[None], _device_map(pc.moment_max)[None]
        if mins.dtype != maxs.dtype:
            mins, maxs = mins.double(), maxs.double()
    out = engine.detect(mins, maxs, float(threshold), int(max_points), patch_size // 2)
    return _to_list(out, 0)
