"""Minimal stand-ins for the parts of ``moekit.tensor`` the layer API touches.

The reference's ``forward_layer`` takes and returns ``tensor.Tensor`` (2-D,
float64, finite-checked; tensor.py:85-127) and raises ``ShapeError``
(tensor.py:47-48). This module keeps those two names so call sites written
against the reference keep working; the arithmetic itself runs in the CUDA
kernels (there is no autodiff tape here: the B200 path is forward-only).
"""

from __future__ import annotations

import numpy as np

__all__ = ["ShapeError", "Tensor", "as_array"]


class ShapeError(ValueError):
    """Raised when operand dimensions do not line up (tensor.py:47-48)."""


class Tensor:
    """Row-major 2-D float64 host matrix (tensor.py:85-127, no tape)."""

    __slots__ = ("value",)

    def __init__(self, value) -> None:
        arr = np.array(value, dtype=np.float64, copy=True)
        if arr.ndim != 2:
            raise ShapeError(f"Tensor must be 2-D, got shape {arr.shape}")
        if arr.size and not np.all(np.isfinite(arr)):
            raise ValueError("Tensor entries must be finite")
        self.value = arr

    @property
    def rows(self) -> int:
        return self.value.shape[0]

    @property
    def cols(self) -> int:
        return self.value.shape[1]

    @property
    def shape(self) -> tuple[int, int]:
        return self.value.shape  # type: ignore[return-value]

    def __repr__(self) -> str:  # pragma: no cover
        return f"Tensor(shape={self.value.shape})"


def as_array(x):
    """Unwrap a Tensor-like (anything with ``.value``, e.g. moekit's Tensor)."""
    return x.value if hasattr(x, "value") and not hasattr(x, "data_ptr") else x
