"""Host-side outlier rejection and affine recovery from matches.

north_star: "the mutual/ratio checks and the FSC/RANSAC outlier stage stay
on the host" and "the recovered affine agrees to within 0.5 px RMSE".  The
reference ships no estimator (ref matcher.py:4-6, SPEC.md:12,429;
parity unpinned), so this is the builder's host stage.  It is applied
identically to the GPU and the CPU-reference match sets: seeded RANSAC over
minimal 3-point samples (vectorised over hypotheses), then least-squares
refits on the inliers until the inlier set stops changing.
"""

from __future__ import annotations

import numpy as np

from .errors import ParameterError


def fit_affine(src, dst) -> np.ndarray:
    """Least-squares 2x3 affine A with dst ~ A @ [x, y, 1] (x, y convention)."""
    src = np.asarray(src, np.float64).reshape(-1, 2)
    dst = np.asarray(dst, np.float64).reshape(-1, 2)
    if len(src) < 3 or len(src) != len(dst):
        raise ParameterError("an affine fit needs >= 3 point pairs")
    X = np.hstack([src, np.ones((len(src), 1))])
    sol, *_ = np.linalg.lstsq(X, dst, rcond=None)
    return sol.T


def apply_affine(a, pts) -> np.ndarray:
    pts = np.asarray(pts, np.float64).reshape(-1, 2)
    a = np.asarray(a, np.float64)
    return pts @ a[:, :2].T + a[:, 2]


def estimate_affine(ref_xy, tgt_xy, threshold: float = 3.0, iters: int = 2000, seed: int = 0,
                    refits: int = 5):
    """RANSAC affine from correspondences ref_xy[i] -> tgt_xy[i].

    Returns (A (2x3) or None, inlier mask).  A hypothesis is scored by its
    number of residuals < threshold (first best on ties); the winner is
    refit by least squares on its inliers, re-scoring after each refit."""
    ref_xy = np.asarray(ref_xy, np.float64).reshape(-1, 2)
    tgt_xy = np.asarray(tgt_xy, np.float64).reshape(-1, 2)
    n = len(ref_xy)
    if n != len(tgt_xy):
        raise ParameterError("ref_xy and tgt_xy must have the same length")
    if n < 3:
        return None, np.zeros(n, bool)
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, n, (iters, 3))
    S = np.concatenate([ref_xy[idx], np.ones((iters, 3, 1))], axis=2)     # (iters, 3, 3)
    D = tgt_xy[idx]                                                        # (iters, 3, 2)
    det = np.linalg.det(S)
    ok = np.abs(det) > 1e-6
    if not ok.any():
        return None, np.zeros(n, bool)
    M = np.linalg.solve(S[ok], D[ok])                                      # (h, 3, 2): [x y 1] @ M = [x' y']
    X = np.hstack([ref_xy, np.ones((n, 1))])
    best, best_cnt = None, -1
    for c0 in range(0, len(M), 256):                                       # bounded memory: 256 x n residuals
        P = np.einsum("nk,hkd->hnd", X, M[c0:c0 + 256])
        cnt = (np.linalg.norm(P - tgt_xy[None], axis=2) < threshold).sum(axis=1)
        j = int(np.argmax(cnt))
        if cnt[j] > best_cnt:
            best, best_cnt = M[c0 + j].T, int(cnt[j])
    inl = np.linalg.norm(apply_affine(best, ref_xy) - tgt_xy, axis=1) < threshold
    for _ in range(refits):
        if inl.sum() < 3:
            return None, inl
        a = fit_affine(ref_xy[inl], tgt_xy[inl])
        new = np.linalg.norm(apply_affine(a, ref_xy) - tgt_xy, axis=1) < threshold
        if np.array_equal(new, inl):
            break
        inl = new
    if inl.sum() < 3:
        return None, inl
    return fit_affine(ref_xy[inl], tgt_xy[inl]), inl


def affine_rmse(a, b, width: int, height: int | None = None, grid: int = 16) -> float:
    """RMSE (px) between two affines over a grid x grid lattice spanning the
    image -- the "recovered affine agrees within 0.5 px" measure."""
    height = width if height is None else height
    ys, xs = np.meshgrid(np.linspace(0, height - 1, grid), np.linspace(0, width - 1, grid), indexing="ij")
    pts = np.stack([xs.ravel(), ys.ravel()], 1)
    d = apply_affine(a, pts) - apply_affine(b, pts)
    return float(np.sqrt(np.mean(np.sum(d * d, axis=1))))


def match_coordinates(result):
    """(ref_xy, tgt_xy) arrays of a PairMatchResult's matches."""
    rk, tk = result.ref.keypoints, result.tgt.keypoints
    ref = np.array([[rk[r].x, rk[r].y] for r, _, _ in result.matches.pairs], np.float64).reshape(-1, 2)
    tgt = np.array([[tk[t].x, tk[t].y] for _, t, _ in result.matches.pairs], np.float64).reshape(-1, 2)
    return ref, tgt
