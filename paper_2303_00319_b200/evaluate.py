"""Ground-truth evaluation of matches, drop-in for ref: pkg/src/rift2/evalbench.py:38-96.

`evaluate` keeps the reference's signature and `EvalReport`; the scoring
itself (transform, residuals, threshold, RMSE) runs in the CUDA kernel
behind `rift2_evaluate` (csrc/evaluate.cu).  `evaluate_batch` scores every
pair of a BatchPipeline step on the device, without building keypoint or
match objects.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import IntegrityError, ParameterError


def _rmse_json(value: float):
    return "∞" if math.isinf(value) else value


@dataclass
class EvalReport:
    """ref: evalbench.py:38-59 (same fields and JSON rendering)."""

    n_correct: int
    rmse: float
    success: bool
    n_matches_total: int
    residual_threshold: float
    timings: dict = field(default_factory=dict)
    descriptor_counts: dict = field(default_factory=dict)

    def to_json_dict(self, with_timings: bool = True) -> dict:
        d = {
            "n_correct": self.n_correct,
            "rmse": _rmse_json(self.rmse),
            "success": self.success,
            "n_matches_total": self.n_matches_total,
            "residual_threshold": self.residual_threshold,
            "descriptor_counts": self.descriptor_counts,
        }
        if with_timings:
            d["timings"] = self.timings
        return d


def transform_row(gt) -> np.ndarray:
    """(R00, R01, R10, R11, t0, t1) of a reference->target transform: a
    RigidTransform-like object (rotation, translation), a generator truth
    with a 2x3 `matrix`, or a 2x3 array."""
    if hasattr(gt, "rotation") and hasattr(gt, "translation"):
        r = np.asarray(gt.rotation, np.float64).reshape(2, 2)
        t = np.asarray(gt.translation, np.float64).reshape(2)
    else:
        m = np.asarray(getattr(gt, "matrix", gt), np.float64)
        if m.shape != (2, 3):
            raise ParameterError(f"ground truth must be 2x3, got {m.shape}")
        r, t = m[:, :2], m[:, 2]
    return np.array([r[0, 0], r[0, 1], r[1, 0], r[1, 1], t[0], t[1]], np.float64)


def evaluate(matches, ref_keypoints, tgt_keypoints, gt, residual_threshold: float = 3.0,
             success_min_matches: int = 10, rmse_cap: float = 20.0, timings: dict | None = None,
             descriptor_counts: dict | None = None) -> EvalReport:
    """ref: evalbench.py:63-96."""
    import torch
    from . import engine
    pairs = matches.pairs
    nr, nt = len(ref_keypoints), len(tgt_keypoints)
    K = max(nr, nt, 1)
    x = np.zeros((2, K), np.int32)
    y = np.zeros((2, K), np.int32)
    for row, kps in enumerate((ref_keypoints, tgt_keypoints)):
        if kps:
            x[row, :len(kps)] = [k.x for k in kps]
            y[row, :len(kps)] = [k.y for k in kps]
    n = len(pairs)
    ids = np.array([(p[0], p[1]) for p in pairs], np.int64).reshape(n, 2)
    if n and (ids.min() < 0 or ids.max() >= 2**31):
        raise IntegrityError(f"match {tuple(ids[np.any((ids < 0) | (ids >= 2**31), axis=1)][0])} "
                             "does not resolve to keypoints")
    rows = np.zeros((2, 1, max(n, 1)), np.int32)
    rows[:, 0, :n] = ids.T
    dev = "cuda"
    kp = dict(x=torch.from_numpy(x).to(dev), y=torch.from_numpy(y).to(dev),
              count=torch.tensor([nr, nt], dtype=torch.int32, device=dev))
    m = dict(ref=torch.from_numpy(rows[0]).to(dev), tgt=torch.from_numpy(rows[1]).to(dev),
             count=torch.tensor([n], dtype=torch.int32, device=dev))
    g = torch.from_numpy(transform_row(gt)[None]).to(dev)
    zero, one = torch.zeros(1, dtype=torch.int32, device=dev), torch.ones(1, dtype=torch.int32, device=dev)
    out = engine.evaluate(kp, zero, one, m, g, residual_threshold, rmse_cap, success_min_matches)
    res = {k: v.cpu().numpy() for k, v in out.items()}
    if res["bad"][0]:
        bad = next((r, t) for r, t, _ in pairs if not (0 <= r < nr and 0 <= t < nt))
        raise IntegrityError(f"match {bad} does not resolve to keypoints")
    return EvalReport(n_correct=int(res["n_correct"][0]), rmse=float(res["rmse"][0]),
                      success=bool(res["success"][0]), n_matches_total=n,
                      residual_threshold=residual_threshold, timings=dict(timings or {}),
                      descriptor_counts=dict(descriptor_counts or {}))


def evaluate_batch(pipe, gts, residual_threshold: float = 3.0, success_min_matches: int = 10,
                   rmse_cap: float = 20.0, out=None) -> dict:
    """Score every pair of a BatchPipeline's last completed step against its
    ground truth (one transform per pair, reference -> target).  Returns
    device tensors n_correct (P,) int32, rmse (P,) float64, success (P,)
    uint8; enqueued on the current stream, no host synchronisation."""
    import torch
    from . import engine
    if torch.is_tensor(gts):
        g = gts.to(device=pipe.dev, dtype=torch.float64)
    else:
        g = torch.from_numpy(np.stack([transform_row(t) for t in gts])).to(pipe.dev)
    if g.shape != (pipe.P, 6):
        raise ParameterError(f"need one transform per pair ({pipe.P}), got {tuple(g.shape)}")
    return engine.evaluate(pipe.k, pipe.rb, pipe.tb, pipe.m, g, residual_threshold, rmse_cap,
                           success_min_matches, out=out)
