"""Phase-congruency data types and parameters, name-compatible with
ref: pkg/src/rift2/loggabor.py:35-119.  The computation itself is the CUDA
filter bank (csrc/fields.cu) reached through pipeline.compute_fields; this
module holds the parameter/result types the callers exchange."""

from __future__ import annotations

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
