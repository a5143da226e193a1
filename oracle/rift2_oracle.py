"""CPU oracle for the RIFT2 feature pipeline -- TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference's hot path
(`/root/reference/pkg/src/rift2`, abbreviated `ref:` below).  It exists so
that the CUDA product path can be checked on the GPU box, where the
reference itself is not present.  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s CPU-baseline / `--impl reference` legs may import it; the
product package never does (it fails loudly when its CUDA library is
missing instead of falling back here).

Parity pin: `tests/test_oracle_golden.py` checks every function below
against golden vectors produced by running the reference itself
(`tests/golden/make_golden.py`, committed together with its outputs).

Each function cites the reference lines it restates.  The arithmetic is
kept operation-for-operation where the reference result is bit-sensitive
(FAST normalisation and scores, the dominant-index ratio test, descriptor
normalisation); elsewhere (FFT library, summation order) agreement is to
float64 rounding.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.fft

# ref: loggabor.py:22-25
EPS = 1e-4
LP_CUTOFF = 0.45
LP_ORDER = 15
# ref: detector.py:21-26  -- radius-3 Bresenham ring, circular order, (dx, dy)
RING16 = (
    (0, -3), (1, -3), (2, -2), (3, -1), (3, 0), (3, 1), (2, 2), (1, 3),
    (0, 3), (-1, 3), (-2, 2), (-3, 1), (-3, 0), (-3, -1), (-2, -2), (-1, -3),
)
ARC = 9


@dataclass(frozen=True)
class Bank:
    """Filter-bank parameters (ref: loggabor.py:35-80, config.py:73-84)."""

    n_scales: int = 4
    n_orient: int = 6
    min_wavelength: float = 3.0
    scale_mult: float = 2.1
    sigma_on_f: float = 0.55
    orientation_spread: float | None = None
    noise_k: float = 2.0
    spread_cutoff: float = 0.5
    spread_gain: float = 10.0

    @property
    def sigma_theta(self) -> float:
        return (math.pi / self.n_orient if self.orientation_spread is None
                else self.orientation_spread)

    def wavelengths(self):
        return self.min_wavelength * self.scale_mult ** np.arange(self.n_scales)

    def angles(self):
        return np.arange(self.n_orient) * np.pi / self.n_orient


def bank_from(cfg) -> Bank:
    """Any object carrying RiftConfig's filter-bank field names."""
    return Bank(*(getattr(cfg, f) for f in (
        "n_scales", "n_orient", "min_wavelength", "scale_mult", "sigma_on_f",
        "orientation_spread", "noise_k", "spread_cutoff", "spread_gain")))


# --------------------------------------------------------------------------
# Filter bank and phase congruency (ref: loggabor.py:122-251, mim.py:43-55)
# --------------------------------------------------------------------------

def transfer(h: int, w: int, p: Bank) -> np.ndarray:
    """(S, O, H, W) log-Gabor transfer functions.  ref: loggabor.py:122-159."""
    fy = np.fft.fftfreq(h).reshape(-1, 1)
    fx = np.fft.fftfreq(w).reshape(1, -1)
    r = np.sqrt(fx * fx + fy * fy)
    r[0, 0] = 1.0
    th = np.arctan2(fy, fx)
    lp = 1.0 / (1.0 + (r / LP_CUTOFF) ** (2 * LP_ORDER))
    denom = 2.0 * np.log(p.sigma_on_f) ** 2
    rad = np.stack([np.exp(-np.log(r * lam) ** 2 / denom) * lp
                    for lam in p.wavelengths()])
    rad[:, 0, 0] = 0.0
    s_t, c_t = np.sin(th), np.cos(th)
    ang = []
    for a in p.angles():
        d = np.abs(np.arctan2(s_t * np.cos(a) - c_t * np.sin(a),
                              c_t * np.cos(a) + s_t * np.sin(a)))
        ang.append(np.exp(-d * d / (2.0 * p.sigma_theta ** 2)))
    g = rad[:, None] * np.stack(ang)[None]
    g[:, :, 0, 0] = 0.0
    return g


def responses(img, p: Bank, workers: int = 1):
    """Complex responses (S, O, H, W).  ref: loggabor.py:162-185."""
    img = np.asarray(img, dtype=np.float64)
    g = transfer(img.shape[0], img.shape[1], p)
    spec = scipy.fft.fft2(img, workers=workers)
    return scipy.fft.ifft2(spec[None, None] * g, axes=(-2, -1), workers=workers)


def phase_congruency(resp: np.ndarray, p: Bank):
    """(a_o, pc_o, moment_max, moment_min).  ref: loggabor.py:193-251."""
    even, odd = resp.real, resp.imag
    amp = np.hypot(even, odd)
    S = resp.shape[0]
    se, so = even.sum(0), odd.sum(0)            # (O, H, W)
    sa, ma = amp.sum(0), amp.max(0)
    xe = np.hypot(se, so) + EPS
    me, mo = se / xe, so / xe
    energy = np.zeros_like(se)
    for s in range(S):
        energy += (even[s] * me + odd[s] * mo
                   - np.abs(even[s] * mo - odd[s] * me))
    # Rayleigh noise floor from the finest scale; ref: loggabor.py:221-228
    tau = np.median(amp[0].reshape(amp.shape[1], -1), axis=1) / math.sqrt(math.log(4.0))
    q = 1.0 / p.scale_mult
    tot = tau * (1 - q ** S) / (1 - q)
    thr = tot * math.sqrt(math.pi / 2) + p.noise_k * tot * math.sqrt((4 - math.pi) / 2)
    energy = np.maximum(energy - thr[:, None, None], 0.0)
    spread = (sa / (ma + EPS) - 1) / max(S - 1, 1)
    wgt = 1.0 / (1.0 + np.exp(p.spread_gain * (p.spread_cutoff - spread)))
    pc = wgt * energy / (sa + EPS)
    ang = p.angles()
    pcc = pc * np.cos(ang)[:, None, None]
    pcs = pc * np.sin(ang)[:, None, None]
    a = (pcc ** 2).sum(0)
    b = 2.0 * (pcc * pcs).sum(0)
    c = (pcs ** 2).sum(0)
    root = np.sqrt(b * b + (a - c) ** 2)
    mmax = 0.5 * (c + a + root)
    mmin = np.maximum(0.5 * (c + a - root), 0.0)
    return sa, pc, mmax, mmin


def max_index_map(a_o: np.ndarray):
    """1-based argmax over orientations (first wins ties) and the max.
    ref: mim.py:43-55."""
    k = np.argmax(a_o, axis=0)
    return (k + 1).astype(np.int32), np.take_along_axis(a_o, k[None], 0)[0]


def fields(img, p: Bank, workers: int = 1):
    """Everything compute_fields produces.  ref: pipeline.py:42-50."""
    a_o, pc, mmax, mmin = phase_congruency(responses(img, p, workers), p)
    mim, amax = max_index_map(a_o)
    return dict(a_o=a_o, pc=pc, moment_max=mmax, moment_min=mmin,
                mim=mim, a_max=amax)


# --------------------------------------------------------------------------
# FAST detection (ref: detector.py:50-155)
# --------------------------------------------------------------------------

KP_DTYPE = np.dtype([("x", np.int32), ("y", np.int32),
                     ("response", np.float64), ("kind", np.int8)])  # kind 0 corner, 1 edge


def normalise(m: np.ndarray) -> np.ndarray:
    """ref: detector.py:80-84."""
    lo, hi = m.min(), m.max()
    if hi - lo <= 0:
        return np.zeros_like(m)
    return (m - lo) / (hi - lo)


def fast_score(n: np.ndarray) -> np.ndarray:
    """Largest threshold at which a 9-of-16 arc passes.  ref: detector.py:50-77."""
    h, w = n.shape
    out = np.zeros((h, w))
    if h <= 6 or w <= 6:
        return out
    ctr = n[3:h - 3, 3:w - 3]
    d = np.stack([n[3 + dy:h - 3 + dy, 3 + dx:w - 3 + dx] - ctr for dx, dy in RING16])
    dd = np.concatenate([d, d[:ARC - 1]], axis=0)       # cyclic extension
    # running minimum over ARC consecutive ring positions, for both signs
    lo = dd[0:16].copy()
    hi = dd[0:16].copy()
    for j in range(1, ARC):
        np.minimum(lo, dd[j:j + 16], out=lo)
        np.maximum(hi, dd[j:j + 16], out=hi)
    bright = lo.max(0)
    dark = -(hi.min(0))
    out[3:h - 3, 3:w - 3] = np.maximum(np.maximum(bright, dark), 0.0)
    return out


def _max3x3(s: np.ndarray) -> np.ndarray:
    """3x3 maximum filter with reflect borders (scipy 'reflect' = edge-mirror)."""
    pad = np.pad(s, 1, mode="symmetric")
    h, w = s.shape
    out = pad[1:h + 1, 1:w + 1].copy()
    for dy in (0, 1, 2):
        for dx in (0, 1, 2):
            np.maximum(out, pad[dy:dy + h, dx:dx + w], out=out)
    return out


def detect_fast(m, thr: float, cap: int, margin: int = 0, kind: int = 0) -> np.ndarray:
    """ref: detector.py:87-113.  Returns a KP_DTYPE array, sorted (-resp, y, x)."""
    m = np.asarray(m, dtype=np.float64)
    s = fast_score(normalise(m))
    keep = (s > thr) & (s == _max3x3(s))
    ys, xs = np.nonzero(keep)
    h, w = m.shape
    if margin > 0:
        ok = (xs >= margin) & (xs <= w - 1 - margin) & (ys >= margin) & (ys <= h - 1 - margin)
        ys, xs = ys[ok], xs[ok]
    r = s[ys, xs]
    order = np.lexsort((xs, ys, -r))[:cap]
    out = np.empty(len(order), KP_DTYPE)
    out["x"], out["y"], out["response"], out["kind"] = xs[order], ys[order], r[order], kind
    return out


_DISK2 = [(dx, dy) for dy in range(-2, 3) for dx in range(-2, 3)
          if (dx, dy) != (0, 0) and dx * dx + dy * dy <= 4]


def merge_radius2(kps: np.ndarray) -> np.ndarray:
    """Greedy suppression within Euclidean 2 px by (-resp, y, x), stable.
    ref: detector.py:116-137 (cKDTree.query_pairs(r=2) is distance <= 2)."""
    n = len(kps)
    if n < 2:
        return kps.copy()
    order = sorted(range(n), key=lambda i: (-kps["response"][i], kps["y"][i], kps["x"][i]))
    at: dict = {}
    for i in range(n):
        at.setdefault((int(kps["x"][i]), int(kps["y"][i])), []).append(i)
    dead = np.zeros(n, bool)
    keep = []
    for i in order:
        if dead[i]:
            continue
        keep.append(i)
        x, y = int(kps["x"][i]), int(kps["y"][i])
        for j in at[(x, y)]:
            dead[j] = True               # coincident points (distance 0)
        for dx, dy in _DISK2:
            for j in at.get((x + dx, y + dy), ()):
                dead[j] = True
    return kps[keep]


def detect_keypoints(mmin, mmax, thr=0.001, cap=5000, patch=96) -> np.ndarray:
    """ref: detector.py:140-155."""
    h, w = np.shape(mmax)
    if h < patch or w < patch:
        raise ValueError("image smaller than the descriptor patch")
    margin = patch // 2
    both = np.concatenate([detect_fast(mmin, thr, cap, margin, 0),
                           detect_fast(mmax, thr, cap, margin, 1)])
    merged = merge_radius2(both)
    # accepted order is already (-resp, y, x); a stable resort keeps it
    idx = sorted(range(len(merged)),
                 key=lambda i: (-merged["response"][i], merged["y"][i], merged["x"][i]))
    return merged[idx][:cap]


# --------------------------------------------------------------------------
# Descriptor (ref: descriptor.py:46-254, mim.py:58-136)
# --------------------------------------------------------------------------

def _snap(v: float) -> float:
    # ref: descriptor.py:58-59
    if abs(v) < 1e-12:
        return 0.0
    if abs(abs(v) - 1) < 1e-12:
        return math.copysign(1.0, v)
    return v


def rotated_offsets(size: int, angle: float):
    """Integer (dx, dy) sample offsets of the rotated grid (size, size).
    ref: descriptor.py:46-82 (nearest neighbour: floor(u + 0.5))."""
    lin = np.arange(size, dtype=np.float64) + 0.5 - size / 2.0
    u, v = np.meshgrid(lin, lin)
    c, s = _snap(math.cos(angle)), _snap(math.sin(angle))
    dx = np.floor(c * u - s * v + 0.5).astype(np.int64)
    dy = np.floor(s * u + c * v + 0.5).astype(np.int64)
    return dx, dy


def patch_at(mim: np.ndarray, x: int, y: int, size: int, angle: float):
    """ref: descriptor.py:85-125 (integer-keypoint paths). None = skip."""
    h, w = mim.shape
    if angle == 0.0:
        x0, y0 = x + 1 - size // 2, y + 1 - size // 2
        if x0 < 0 or y0 < 0 or x0 + size > w or y0 + size > h:
            return None
        return mim[y0:y0 + size, x0:x0 + size]
    dx, dy = rotated_offsets(size, angle)
    if x + dx.min() < 0 or x + dx.max() >= w or y + dy.min() < 0 or y + dy.max() >= h:
        return None
    return mim[y + dy, x + dx]


def dominant(hist, ratio: float = 0.8):
    """ref: mim.py:69-91."""
    hist = np.asarray(hist, dtype=np.float64)
    n = len(hist)
    pk = int(np.argmax(hist))
    rest = hist.copy()
    rest[pk] = -np.inf
    rv = rest.max()
    picks = [pk + 1]
    if rv >= ratio * hist[pk]:
        cand = np.flatnonzero(rest == rv)
        picks.append(int(cand[np.argmin((cand - pk) % n)]) + 1)
    return picks


def recode_values(v: np.ndarray, dom: int, n: int) -> np.ndarray:
    """ref: mim.py:97-125 ('recode' table: v>=s -> v-s+1 else v+n-s+1)."""
    return np.where(v >= dom, v - dom + 1, v + n - dom + 1)


def cell_counts(patch: np.ndarray, grid: int, n: int) -> np.ndarray:
    """Integer per-cell index histogram, (grid*grid*n,) int64.
    ref: descriptor.py:131-164 (bincount of cell*n - 1 + value)."""
    size = patch.shape[0]
    cs = size // grid
    cell = (np.arange(size) // cs)
    cid = cell[:, None] * grid + cell[None, :]
    return np.bincount((cid * n - 1 + patch).ravel(), minlength=grid * grid * n)


def unit(counts: np.ndarray) -> np.ndarray:
    """ref: descriptor.py:161-164 (np.linalg.norm then divide)."""
    v = counts.astype(np.float64)
    return v / np.linalg.norm(v)


DESC_DTYPE_FIELDS = ("counts", "kp", "variant")


def describe_rift2(mim, kps, size=96, grid=6, ratio=0.8, rotate=True, n_orient=6):
    """ref: descriptor.py:179-216.  Returns (counts (D, grid*grid*n) int64,
    kp ids (D,), variants (D,), skipped)."""
    step = math.pi / n_orient
    out_c, out_k, out_v = [], [], []
    skipped = 0
    for i, (x, y) in enumerate(zip(np.asarray(kps["x"]), np.asarray(kps["y"]))):
        base = patch_at(mim, int(x), int(y), size, 0.0)
        if base is None:
            skipped += 1
            continue
        hist = np.bincount(base.ravel(), minlength=n_orient + 1)[1:]
        for dom in dominant(hist, ratio):
            pt = base
            if rotate and dom != 1:
                pt = patch_at(mim, int(x), int(y), size, (dom - 1) * step)
                if pt is None:
                    skipped += 1
                    continue
            out_c.append(cell_counts(recode_values(pt, dom, n_orient), grid, n_orient))
            out_k.append(i)
            out_v.append(dom)
    dim = grid * grid * n_orient
    return (np.array(out_c, dtype=np.int64).reshape(-1, dim),
            np.array(out_k, dtype=np.int64), np.array(out_v, dtype=np.int64), skipped)


def describe_ring(mim, kps, size=96, grid=6, n_orient=6):
    """ref: descriptor.py:219-236 (cyclic_shift table (v - s) % n + 1)."""
    out_c, out_k, out_v = [], [], []
    skipped = 0
    for i, (x, y) in enumerate(zip(np.asarray(kps["x"]), np.asarray(kps["y"]))):
        base = patch_at(mim, int(x), int(y), size, 0.0)
        if base is None:
            skipped += 1
            continue
        for layer in range(1, n_orient + 1):
            out_c.append(cell_counts((base - layer) % n_orient + 1, grid, n_orient))
            out_k.append(i)
            out_v.append(layer)
    dim = grid * grid * n_orient
    return (np.array(out_c, dtype=np.int64).reshape(-1, dim),
            np.array(out_k, dtype=np.int64), np.array(out_v, dtype=np.int64), skipped)


def describe_plain(mim, kps, size=96, grid=6, n_orient=6):
    """ref: descriptor.py:239-254."""
    out_c, out_k = [], []
    skipped = 0
    for i, (x, y) in enumerate(zip(np.asarray(kps["x"]), np.asarray(kps["y"]))):
        base = patch_at(mim, int(x), int(y), size, 0.0)
        if base is None:
            skipped += 1
            continue
        out_c.append(cell_counts(base, grid, n_orient))
        out_k.append(i)
    dim = grid * grid * n_orient
    return (np.array(out_c, dtype=np.int64).reshape(-1, dim),
            np.array(out_k, dtype=np.int64), np.ones(len(out_k), np.int64), skipped)


# --------------------------------------------------------------------------
# Matching (ref: matcher.py:67-148)
# --------------------------------------------------------------------------

def match_nn(ref_vec, ref_kp, tgt_vec, tgt_kp, block: int = 1024):
    """Nearest reference keypoint for every target keypoint.

    ref_vec/tgt_vec are unit float64 rows; *_kp their keypoint ids.  Key per
    descriptor pair is |r|^2 - 2 r.t (ref: matcher.py:125-129), minimised
    over both variant groups, first index on ties; exact distance of the
    winner from difference vectors (ref: matcher.py:137-141).  Returns an
    (N, 3) list of (ref_id, tgt_id, dist) sorted by (dist, ref, tgt) and the
    distance-evaluation count.
    """
    ro = np.argsort(ref_kp, kind="stable")
    to = np.argsort(tgt_kp, kind="stable")
    R, rk = np.asarray(ref_vec)[ro], np.asarray(ref_kp)[ro]
    T, tk = np.asarray(tgt_vec)[to], np.asarray(tgt_kp)[to]
    r_ids, r_first = np.unique(rk, return_index=True)
    t_ids, t_first = np.unique(tk, return_index=True)
    r_grp = np.searchsorted(r_ids, rk)
    t_grp = np.searchsorted(t_ids, tk)
    rsq = (R * R).sum(1)
    best = np.empty(len(t_ids), np.int64)
    for g0 in range(0, len(t_ids), block):
        g1 = min(g0 + block, len(t_ids))
        rows = np.flatnonzero((t_grp >= g0) & (t_grp < g1))
        key = rsq[:, None] - 2.0 * (R @ T[rows].T)          # (nR, nrows)
        per_rk = np.full((len(r_ids), len(rows)), np.inf)
        np.minimum.at(per_rk, r_grp, key)
        per_g = np.full((len(r_ids), g1 - g0), np.inf)
        np.minimum.at(per_g.T, t_grp[rows] - g0, per_rk.T)
        best[g0:g1] = np.argmin(per_g, axis=0)
    pairs = []
    for g in range(len(t_ids)):
        rr = R[r_grp == best[g]]
        tt = T[t_grp == g]
        d = rr[:, None, :] - tt[None, :, :]
        pairs.append((int(r_ids[best[g]]), int(t_ids[g]),
                      float(np.sqrt((d * d).sum(-1).min()))))
    pairs.sort(key=lambda p: (p[2], p[0], p[1]))
    return pairs, len(R) * len(T)


# ---------------------------------------------------------------- evaluation
def evaluate(ref_xy, tgt_xy, pairs, gt_row, thr: float = 3.0, min_matches: int = 10, cap: float = 20.0):
    """ref: evalbench.py:63-96 -- (n_correct, rmse, success).  gt_row =
    (R00, R01, R10, R11, t0, t1); p' = p @ R^T + t (ref: imaging.py:71-74).
    Raises IndexError where the reference raises IntegrityError."""
    ref_xy = np.asarray(ref_xy, np.float64).reshape(-1, 2)
    tgt_xy = np.asarray(tgt_xy, np.float64).reshape(-1, 2)
    pairs = np.asarray(pairs, np.int64).reshape(-1, 2)
    if len(pairs) and (pairs.min() < 0 or pairs[:, 0].max() >= len(ref_xy) or pairs[:, 1].max() >= len(tgt_xy)):
        raise IndexError("match does not resolve to keypoints")
    if not len(pairs):
        return 0, math.inf, 0 >= min_matches
    rot = np.array(gt_row[:4], np.float64).reshape(2, 2)
    res = np.linalg.norm(ref_xy[pairs[:, 0]] @ rot.T + np.array(gt_row[4:], np.float64) - tgt_xy[pairs[:, 1]],
                         axis=1)
    ok = res < thr
    n = int(ok.sum())
    rmse = min(float(np.sqrt(np.mean(res[ok] ** 2))), cap) if n else math.inf
    return n, rmse, n >= min_matches
