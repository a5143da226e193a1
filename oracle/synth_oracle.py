"""CPU checker for the on-device target synthesis.

TEST INFRASTRUCTURE ONLY: imported by tests/ as the checker of
`rift2_synth_targets` (csrc/synth.cu); never by the product package.

The reference ships no BASELINE generator; the warp follows
ref: pkg/src/rift2/imaging.py:208-247 (`warp_rigid`: output p samples the
source bilinearly at T^-1(p), zero outside, exactly-on-grid samples on the
far edges kept), generalised to a similarity, followed by the BASELINE
radiometry (inversion, gamma, multiplicative Gamma(L, 1/L) speckle, min-max
renormalisation).  The speckle uses a counter-based generator so the device
and this checker draw the same numbers:

* Philox4x32-10 (Salmon et al., "Parallel random numbers: as easy as 1, 2,
  3", SC'11): 10 rounds of the two 32x32->64 multiplies with constants
  0xD2511F53 / 0xCD9E8D57 and the Weyl key bumps 0x9E3779B9 / 0xBB67AE85;
  pinned by its published all-zero answer in tests/test_synth_host.py;
* counter (pixel index lo, pixel index hi, image index, draw pair j), key
  (seed lo, seed hi); one block gives two 53-bit uniforms in (0, 1];
* Gamma(L, 1/L) for integer L as the mean of L unit exponentials
  -log(u) (the Erlang construction).
"""

from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 on uint32 arrays (broadcasting)."""
    c0, c1, c2, c3 = (np.asarray(v, np.uint32) for v in (c0, c1, c2, c3))
    k0, k1 = np.asarray(k0, np.uint32), np.asarray(k1, np.uint32)
    with np.errstate(over="ignore"):
        for r in range(10):
            p0 = c0.astype(np.uint64) * M0
            p1 = c2.astype(np.uint64) * M1
            hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & MASK).astype(np.uint32)
            hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & MASK).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            if r < 9:
                k0 = (k0 + W0).astype(np.uint32)
                k1 = (k1 + W1).astype(np.uint32)
    return c0, c1, c2, c3


def uniforms53(a, b):
    """(0, 1] double from two 32-bit words: ((a >> 5) * 2^26 + (b >> 6) + 1) * 2^-53."""
    m = (np.asarray(a, np.uint64) >> np.uint64(5)) * np.uint64(1 << 26) + (np.asarray(b, np.uint64) >> np.uint64(6))
    return (m + np.uint64(1)).astype(np.float64) * 2.0 ** -53


def speckle(h: int, w: int, image: int, looks: int, seed: int) -> np.ndarray:
    """Gamma(looks, 1/looks) field of one image (float64, (h, w))."""
    idx = np.arange(h * w, dtype=np.uint64)
    c0 = (idx & MASK).astype(np.uint32)
    c1 = (idx >> np.uint64(32)).astype(np.uint32)
    k0, k1 = np.uint32(seed & 0xFFFFFFFF), np.uint32((seed >> 32) & 0xFFFFFFFF)
    s = np.zeros(h * w)
    for j in range((looks + 1) // 2):
        r0, r1, r2, r3 = philox4x32_10(c0, c1, np.uint32(image), np.uint32(j), k0, k1)
        s = s + -np.log(uniforms53(r0, r1))
        if 2 * j + 1 < looks:
            s = s + -np.log(uniforms53(r2, r3))
    return (s / looks).reshape(h, w)


def warp(img: np.ndarray, inv: np.ndarray) -> np.ndarray:
    """Bilinear warp, `inv` the 2x3 inverse map (output -> source), float64,
    the operation order of ref: imaging.py:225-246."""
    h, w = img.shape
    xs, ys = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    sx = inv[0, 0] * xs + inv[0, 1] * ys + inv[0, 2]
    sy = inv[1, 0] * xs + inv[1, 1] * ys + inv[1, 2]
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


def synth_target(img: np.ndarray, inv: np.ndarray, inverted: bool, gamma: float, looks: int, seed: int,
                 image: int = 0) -> np.ndarray:
    """Target image (float64) of one pair: warp, inversion, gamma, speckle,
    min-max renormalisation (the BASELINE generator's radiometry)."""
    v = warp(np.asarray(img, np.float64), np.asarray(inv, np.float64))
    if inverted:
        v = 1.0 - v
    v = np.clip(v, 0.0, 1.0) ** gamma
    if looks:
        v = v * speckle(v.shape[0], v.shape[1], image, looks, seed)
    return (v - v.min()) / max(v.max() - v.min(), 1e-12)
