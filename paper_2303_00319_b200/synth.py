"""Seeded synthetic image pairs standing in for the paper's datasets.

The LNIFT SAR-optical / infrared-optical sets the paper measures on are not
available here, and the reference's own `synthetic.py` does
not contain the BASELINE.json generator, so this module is a
builder-written restatement of the BASELINE.json config text:

* image 1: anisotropic Gaussian blobs (sigma 2-20 px, x4 for 4096^2) plus
  band-limited white noise (all FFT bins with radial frequency >= 0.2
  cyc/px zeroed), min-max normalised to [0, 1];
* image 2: image 1 under a similarity p' = s R (p - c) + c + t about the
  centre c (bilinear, zero fill, `warp_rigid` semantics of
  ref: imaging.py:208-247), then inversion (p = 0.5), gamma in [0.4, 2.5],
  multiplicative Gamma(L, 1/L) speckle, re-normalised to [0, 1].

Everything is numpy float64 on the host and deterministic per seed.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class PairTruth:
    """Ground truth of one generated pair (maps reference -> target)."""

    theta_deg: float
    scale: float
    translation: tuple
    inverted: bool
    gamma: float
    looks: int
    size: int
    matrix: np.ndarray = field(default=None)   # 2x3 affine, (x, y) convention

    def apply(self, pts) -> np.ndarray:
        pts = np.asarray(pts, dtype=np.float64).reshape(-1, 2)
        return pts @ self.matrix[:, :2].T + self.matrix[:, 2]


def blob_field(size: int, seed: int, n_blobs: int = 200, sigma_scale: float = 1.0,
               noise_weight: float = 0.5, f_cut: float = 0.2) -> np.ndarray:
    """Image 1 of the BASELINE generator (see module docstring)."""
    rng = np.random.default_rng(seed)
    img = np.zeros((size, size))
    for _ in range(n_blobs):
        cx, cy = rng.uniform(0, size, 2)
        sx, sy = rng.uniform(2.0, 20.0, 2) * sigma_scale
        phi = rng.uniform(0, math.pi)
        amp = rng.uniform(-1.0, 1.0)
        ext = int(math.ceil(4.0 * max(sx, sy)))
        x0, x1 = max(int(cx) - ext, 0), min(int(cx) + ext + 1, size)
        y0, y1 = max(int(cy) - ext, 0), min(int(cy) + ext + 1, size)
        if x0 >= x1 or y0 >= y1:
            continue
        ys, xs = np.mgrid[y0:y1, x0:x1].astype(np.float64)
        dx, dy = xs - cx, ys - cy
        u = math.cos(phi) * dx + math.sin(phi) * dy
        v = -math.sin(phi) * dx + math.cos(phi) * dy
        img[y0:y1, x0:x1] += amp * np.exp(-0.5 * ((u / sx) ** 2 + (v / sy) ** 2))
    white = rng.standard_normal((size, size))
    spec = np.fft.fft2(white)
    f = np.fft.fftfreq(size)
    spec[np.hypot(f[:, None], f[None, :]) >= f_cut] = 0.0
    noise = np.fft.ifft2(spec).real
    noise /= max(noise.std(), 1e-12)
    img /= max(img.std(), 1e-12)
    img = img + noise_weight * noise
    return (img - img.min()) / (img.max() - img.min())


def blob_params(size: int, seed: int, n_blobs: int = 200, sigma_scale: float = 1.0):
    """The blob draws of blob_field, in its order, as rift2_synth_blobs rows
    (cx, cy, sx, sy, cos phi, sin phi, amp, x0, x1, y0, y1); returns the rows
    and the generator positioned at the white-noise draw."""
    rng = np.random.default_rng(seed)
    rows = np.zeros((n_blobs, 11))
    for i in range(n_blobs):
        cx, cy = rng.uniform(0, size, 2)
        sx, sy = rng.uniform(2.0, 20.0, 2) * sigma_scale
        phi = rng.uniform(0, math.pi)
        amp = rng.uniform(-1.0, 1.0)
        ext = int(math.ceil(4.0 * max(sx, sy)))
        x0, x1 = max(int(cx) - ext, 0), min(int(cx) + ext + 1, size)
        y0, y1 = max(int(cy) - ext, 0), min(int(cy) + ext + 1, size)
        rows[i] = (cx, cy, sx, sy, math.cos(phi), math.sin(phi), amp, x0, x1, y0, y1)
    return rows, rng


def image1_device(n_images: int, size: int, seed0: int = 0, noise: str = "device", sigma_scale: float | None = None,
                  noise_weight: float = 0.5, f_cut: float = 0.2, noise_seed: int | None = None):
    """Image 1 of the generator for seeds seed0.. on the GPU -> (n, size,
    size) float64 CUDA tensor.  The blobs are rift2_synth_blobs on the host's
    own draws (blob_params); the white noise is the host's standard_normal
    draw ("host": the same image as blob_field up to float32 FFT rounding) or
    Philox normals on the device ("device", key noise_seed, default seed0:
    a different but equally distributed noise field, no host work); the
    band-limit is rift2_apply_bank with a 0/1 mask of radial frequency <
    f_cut; then blob_field's normalisation."""
    import torch
    from . import engine
    if sigma_scale is None:
        sigma_scale = 4.0 if size >= 4096 else 1.0
    rows, hostnoise = [], []
    for i in range(n_images):
        r, rng = blob_params(size, seed0 + i, sigma_scale=sigma_scale)
        rows.append(r)
        if noise == "host":
            hostnoise.append(rng.standard_normal((size, size)).astype(np.float32))
    img = engine.synth_blobs(torch.from_numpy(np.stack(rows)).cuda(), size, size)
    if noise == "host":
        white = torch.from_numpy(np.stack(hostnoise)).cuda()
    else:
        white = engine.synth_normals(seed0 if noise_seed is None else noise_seed, 0, n_images, size * size)
        white = white.view(n_images, size, size)
    f = np.fft.fftfreq(size)
    mask = torch.from_numpy((np.hypot(f[:, None], f[None, :]) < f_cut).astype(np.float32)[None, None]).cuda()
    for i in range(n_images):
        even, _, _ = engine.apply_bank(white[i].contiguous(), mask)
        nz = even[0, 0].double()
        nz = nz / torch.clamp(nz.std(unbiased=False), min=1e-12)
        im = img[i]
        im = im / torch.clamp(im.std(unbiased=False), min=1e-12)
        im = im + noise_weight * nz
        img[i] = (im - im.min()) / (im.max() - im.min())
    return img


def similarity(size: int, theta_deg: float, scale: float, t) -> np.ndarray:
    """2x3 matrix of p' = s R (p - c) + c + t, c the image centre."""
    c = (size - 1) / 2.0
    th = math.radians(theta_deg)
    co, si = math.cos(th), math.sin(th)
    # snap quarter turns like ref: imaging.py:61-63
    co = 0.0 if abs(co) < 1e-15 else (math.copysign(1.0, co) if abs(abs(co) - 1) < 1e-15 else co)
    si = 0.0 if abs(si) < 1e-15 else (math.copysign(1.0, si) if abs(abs(si) - 1) < 1e-15 else si)
    a = scale * np.array([[co, -si], [si, co]])
    off = np.array([c, c]) + np.asarray(t, dtype=np.float64) - a @ np.array([c, c])
    return np.concatenate([a, off[:, None]], axis=1)


def warp(img: np.ndarray, m: np.ndarray) -> np.ndarray:
    """Output p samples img at m^-1(p), bilinear, zero outside
    (ref: imaging.py:208-247 semantics, generalised to a similarity)."""
    h, w = img.shape
    inv = inverse_map(m)
    a_inv, t_inv = inv[:, :2], inv[:, 2]
    xs, ys = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    sx = a_inv[0, 0] * xs + a_inv[0, 1] * ys + t_inv[0]
    sy = a_inv[1, 0] * xs + a_inv[1, 1] * ys + t_inv[1]
    x0 = np.floor(sx).astype(np.int64)
    y0 = np.floor(sy).astype(np.int64)
    fx, fy = sx - x0, sy - y0
    out = np.zeros((h, w))
    ok = (x0 >= 0) & (x0 < w - 1) & (y0 >= 0) & (y0 < h - 1)
    on = (fx == 0) & (fy == 0) & (x0 >= 0) & (x0 < w) & (y0 >= 0) & (y0 < h)
    xv, yv, fxv, fyv = x0[ok], y0[ok], fx[ok], fy[ok]
    out[ok] = (img[yv, xv] * (1 - fxv) * (1 - fyv) + img[yv, xv + 1] * fxv * (1 - fyv)
               + img[yv + 1, xv] * (1 - fxv) * fyv + img[yv + 1, xv + 1] * fxv * fyv)
    edge = on & ~ok
    out[edge] = img[y0[edge], x0[edge]]
    return out


def _pair_draws(size: int, seed: int, theta_deg, scale_jitter: float, looks):
    """The per-pair parameter draws of make_pair, in its order; returns the
    truth and the generator (positioned at the speckle draws)."""
    rng = np.random.default_rng(10_000 + seed)
    theta = float(rng.uniform(0.0, 360.0)) if theta_deg is None else float(theta_deg)
    scale = float(rng.uniform(1.0 - scale_jitter, 1.0 + scale_jitter)) if scale_jitter else 1.0
    t = tuple(float(v) for v in rng.uniform(-20.0, 20.0, 2))
    m = similarity(size, theta, scale, t)
    inverted = bool(rng.uniform() < 0.5)
    gamma = float(rng.uniform(0.4, 2.5))
    return PairTruth(theta, scale, t, inverted, gamma, looks or 0, size, m), rng


def inverse_map(m: np.ndarray) -> np.ndarray:
    """2x3 target->source map of a 2x3 source->target affine, as `warp` forms it."""
    a_inv = np.linalg.inv(m[:, :2])
    return np.concatenate([a_inv, (-a_inv @ m[:, 2])[:, None]], axis=1)


def make_pair(size: int = 1024, seed: int = 0, theta_deg: float | None = None,
              scale_jitter: float = 0.0, looks: int | None = 4,
              sigma_scale: float | None = None, radiometric: bool = True):
    """(image1, image2, truth) per the BASELINE.json generator, float64."""
    if sigma_scale is None:
        sigma_scale = 4.0 if size >= 4096 else 1.0
    img1 = blob_field(size, seed, sigma_scale=sigma_scale)
    truth, rng = _pair_draws(size, seed, theta_deg, scale_jitter, looks)
    img2 = warp(img1, truth.matrix)
    inverted, gamma = truth.inverted, truth.gamma
    if radiometric:
        if inverted:
            img2 = 1.0 - img2
        img2 = np.clip(img2, 0.0, 1.0) ** gamma
        if looks:
            img2 = img2 * rng.gamma(float(looks), 1.0 / looks, img2.shape)
        img2 = (img2 - img2.min()) / max(img2.max() - img2.min(), 1e-12)
    return img1, img2, truth


def make_batch(n_pairs: int, size: int = 1024, seed0: int = 0, dtype=np.float32, **kw):
    """(2*n_pairs, size, size) stack [ref0, tgt0, ref1, tgt1, ...] + truths."""
    out = np.empty((2 * n_pairs, size, size), dtype=dtype)
    truths = []
    for i in range(n_pairs):
        a, b, tr = make_pair(size, seed0 + i, **kw)
        out[2 * i], out[2 * i + 1] = a, b
        truths.append(tr)
    return out, truths


def make_batch_device(n_pairs: int, size: int = 1024, seed0: int = 0, device="cuda", speckle_seed: int | None = None,
                      theta_deg: float | None = None, scale_jitter: float = 0.0, looks: int | None = 4,
                      sigma_scale: float | None = None, radiometric: bool = True, image1: str = "host"):
    """make_batch with the target side synthesised on the GPU
    (rift2_synth_targets); image 1 from the host generator (image1="host"),
    or on the GPU (image1="device": image1_device with Philox white noise;
    "device_hostnoise": the host's noise draw); the per-pair draws (hence the
    truths) are the host generator's; the warp, inversion, gamma and renormalisation
    match make_pair to float32 rounding (pow on the device is within 2 ulp);
    the speckle is drawn from Philox4x32-10 (key speckle_seed, default
    seed0; counter word 2 = pair index) instead of numpy's stream.
    Returns the (2 * n_pairs, size, size) float32 CUDA stack and the truths."""
    import torch
    from . import engine
    if sigma_scale is None:
        sigma_scale = 4.0 if size >= 4096 else 1.0
    params = np.zeros((n_pairs, 8))
    truths = []
    if image1 == "host":
        src = np.empty((n_pairs, size, size))
        for i in range(n_pairs):
            src[i] = blob_field(size, seed0 + i, sigma_scale=sigma_scale)
    for i in range(n_pairs):
        tr, _ = _pair_draws(size, seed0 + i, theta_deg, scale_jitter, looks)
        params[i, :6] = inverse_map(tr.matrix).ravel()
        params[i, 6] = tr.gamma
        params[i, 7] = (1 if tr.inverted else 0) | (2 if radiometric else 0)
        truths.append(tr)
    out = torch.empty((2 * n_pairs, size, size), dtype=torch.float32, device=device)
    d_src = torch.from_numpy(src).to(device) if image1 == "host" else \
        image1_device(n_pairs, size, seed0, noise="host" if image1 == "device_hostnoise" else "device",
                      sigma_scale=sigma_scale)
    d_par = torch.from_numpy(params).to(device)
    d_looks = torch.full((n_pairs,), int(looks or 0), dtype=torch.int32, device=device)
    engine.synth_targets(d_src, d_par, d_looks, seed0 if speckle_seed is None else speckle_seed, out[1::2],
                         src_copy=out[0::2])
    return out, truths
