"""Maximum index map type, name-compatible with ref: pkg/src/rift2/mim.py:21-40.
The map itself is produced by the filter-bank kernel (csrc/fields.cu, the
argmax over orientation amplitude sums of ref: mim.py:43-55)."""

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
