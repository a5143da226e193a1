"""Log-Gabor filter bank and phase congruency, drop-in for
ref: pkg/src/rift2/loggabor.py.  The pipeline path is the fused CUDA filter
bank (csrc/fields.cu, rift2_fields) reached through pipeline.compute_fields;
the reference's step-by-step entry points (build_filter_bank, apply_bank,
orientation_amplitudes, phase_congruency_moments) run on their own CUDA
kernels of the same library (rift2_filter_bank, rift2_apply_bank,
rift2_orientation_amplitudes, rift2_pc_moments)."""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from .errors import ParameterError

EPSILON = 1e-4
LOWPASS_CUTOFF = 0.45
LOWPASS_ORDER = 15


@dataclass(frozen=True)
class BankParams:
    """Filter-bank tunables (ref: loggabor.py:35-80), same validation."""

    n_scales: int = 4
    n_orient: int = 6
    min_wavelength: float = 3.0
    scale_mult: float = 2.1
    sigma_on_f: float = 0.55
    orientation_spread: float | None = None
    noise_k: float = 2.0
    spread_cutoff: float = 0.5
    spread_gain: float = 10.0

    def __post_init__(self):
        if self.n_scales < 1:
            raise ParameterError("n_scales must be >= 1")
        if self.n_orient < 2:
            raise ParameterError("n_orient must be >= 2")
        if self.min_wavelength < 2:
            raise ParameterError("min_wavelength must be >= 2")
        if self.scale_mult <= 1:
            raise ParameterError("scale_mult must be > 1")
        if not 0 < self.sigma_on_f < 1:
            raise ParameterError("sigma_on_f must be in (0, 1)")

    @property
    def angular_sigma(self) -> float:
        return self.orientation_spread if self.orientation_spread is not None else np.pi / self.n_orient

    def wavelengths(self) -> np.ndarray:
        return self.min_wavelength * self.scale_mult ** np.arange(self.n_scales)

    def orientation_angles(self) -> np.ndarray:
        return np.arange(self.n_orient) * np.pi / self.n_orient


@dataclass(frozen=True)
class PCField:
    """Per-orientation amplitude sums, phase congruency and moment maps
    (ref: loggabor.py:106-119).  Maps produced by compute_fields are
    read-only and keep a device copy (_devcache) that detect_keypoints reuses."""

    a_o: np.ndarray
    pc_per_orientation: np.ndarray
    moment_max: np.ndarray
    moment_min: np.ndarray

    @property
    def shape(self):
        return self.moment_max.shape


def fft_workers(threads: int = 0) -> int:
    """ref: loggabor.py:28-32 (worker count of the reference's CPU FFTs; kept
    for API compatibility -- the transforms here run on the GPU)."""
    if threads and threads > 0:
        return threads
    return os.cpu_count() or 1


@dataclass(frozen=True)
class FilterBank:
    """Transfer functions (n_scales, n_orient, height, width) float64
    (ref: loggabor.py:83-92)."""

    transfer: np.ndarray
    params: BankParams

    @property
    def shape(self):
        return self.transfer.shape[2], self.transfer.shape[3]


@dataclass(frozen=True)
class ConvolutionStack:
    """Even / odd quadrature responses and their amplitude per scale and
    orientation, (n_scales, n_orient, height, width) (ref: loggabor.py:95-103)."""

    even: np.ndarray
    odd: np.ndarray
    amplitude: np.ndarray
    params: BankParams


def build_filter_bank(width: int, height: int, params: BankParams | None = None) -> FilterBank:
    """ref: loggabor.py:131-159 -- computed by the rift2_filter_bank kernel in
    float64 with the reference's formulas."""
    from . import engine
    params = params or BankParams()
    if width < 16 or height < 16:
        raise ParameterError("filter bank needs width and height >= 16")
    t = engine.filter_bank(int(height), int(width), params)
    return FilterBank(transfer=t.cpu().numpy(), params=params)


def apply_bank(img, bank: FilterBank, threads: int = 0) -> ConvolutionStack:
    """ref: loggabor.py:162-185 -- the given bank applied by the CUDA FFT
    passes (rift2_apply_bank, float32 arithmetic; float64 results)."""
    import torch
    from . import engine
    from .pipeline import check_image
    arr = check_image(img)
    if arr.shape != bank.shape:
        raise ParameterError(f"image shape {arr.shape} does not match bank shape {bank.shape}")
    image = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).cuda()
    transfer = torch.from_numpy(np.ascontiguousarray(bank.transfer, dtype=np.float32)).cuda()
    even, odd, amp = engine.apply_bank(image, transfer)
    return ConvolutionStack(even=even.double().cpu().numpy(), odd=odd.double().cpu().numpy(),
                            amplitude=amp.double().cpu().numpy(), params=bank.params)


def orientation_amplitudes(stack: ConvolutionStack) -> np.ndarray:
    """ref: loggabor.py:188-190 -- sum over scales (rift2_orientation_amplitudes, float64)."""
    import torch
    from . import engine
    amp = np.asarray(stack.amplitude, dtype=np.float64)
    if amp.ndim != 4:
        raise ParameterError(f"expected a (scales, orientations, h, w) stack, got shape {amp.shape}")
    out = engine.orientation_amplitudes(torch.from_numpy(np.ascontiguousarray(amp)).cuda())
    return out.cpu().numpy()


def phase_congruency_moments(stack: ConvolutionStack, params: BankParams | None = None) -> PCField:
    """ref: loggabor.py:193-251 -- per-orientation phase congruency and the
    moment maps from a response stack (rift2_pc_moments, float32 arithmetic,
    exact median noise floor)."""
    import torch
    from . import engine
    params = params or stack.params
    amp = np.asarray(stack.amplitude)
    if amp.ndim != 4 or amp.shape[0] != params.n_scales or amp.shape[1] != params.n_orient:
        raise ParameterError(f"stack shape {amp.shape} does not match the bank parameters")
    planes = [torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda() for a in (stack.even, stack.odd, amp)]
    out = engine.pc_moments(*planes, params)
    return PCField(a_o=orientation_amplitudes(stack), pc_per_orientation=out["pc"].double().cpu().numpy(),
                   moment_max=out["mmax"].double().cpu().numpy(), moment_min=out["mmin"].double().cpu().numpy())
