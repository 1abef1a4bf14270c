"""Bound configuration objects of the reference, mirrored for the drop-in API.

``RadiusConfig`` / ``CellBounds`` keep the reference's field names, defaults,
validation and messages (colbandit/bounds.py:112-191). The interval
arithmetic itself (hard bounds, radius, decision interval, score proxy —
bounds.py:72-263) runs inside the bandit kernel (csrc/bandit.cu
``row_interval``); only ``log_term`` is evaluated here, on the host, with
``math.log`` exactly as the reference does (bounds.py:138-143), because a
device ``log`` may differ in the last ulp.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

UNION_MODES = ("per-document", "per-document-and-size")

__all__ = ["RadiusConfig", "CellBounds", "UNION_MODES", "fp_correction"]


@dataclass(frozen=True)
class RadiusConfig:
    alpha_ef: float = 1.0
    delta: float = 0.01
    c: float = 1.0
    union_mode: str = "per-document"

    def __post_init__(self) -> None:
        if not 0.0 < self.alpha_ef <= 1.0:
            raise ValueError(f"alpha_ef must be in (0, 1], got {self.alpha_ef}")
        if not 0.0 < self.delta < 1.0:
            raise ValueError(f"delta must be in (0, 1), got {self.delta}")
        if self.c <= 0.0:
            raise ValueError(f"c must be positive, got {self.c}")
        if self.union_mode not in UNION_MODES:
            raise ValueError(f"union_mode must be one of {UNION_MODES}, got {self.union_mode!r}")

    def log_term(self, n_rows: int, n_cols: int) -> float:
        """max(log(c N / delta [* T]), 0) — bounds.py:138-143."""
        arg = self.c * n_rows / self.delta
        if self.union_mode == "per-document-and-size":
            arg *= n_cols
        return max(math.log(arg), 0.0)


def fp_correction(n: int, n_cols: int) -> float:
    """Finite-population factor rho_n (bounds.py:97-109); the kernel evaluates the same expression."""
    n = int(n)
    if not 1 <= n <= n_cols:
        raise ValueError(f"fp_correction needs 1 <= n <= {n_cols}, got n={n}")
    if 2 * n <= n_cols:
        return 1.0 - (n - 1) / n_cols
    return (1.0 - n / n_cols) * (1.0 + 1.0 / n)


class CellBounds:
    """Per-cell support bounds ``lo[i, t] <= H[i, t] <= hi[i, t]`` (bounds.py:161-191)."""

    def __init__(self, lo, hi):
        lo = np.asarray(lo, dtype=np.float64)
        hi = np.asarray(hi, dtype=np.float64)
        if lo.ndim != 2 or lo.shape != hi.shape:
            raise ValueError(f"bound arrays must share a 2-D shape, got {lo.shape} and {hi.shape}")
        if not (np.all(np.isfinite(lo)) and np.all(np.isfinite(hi))):
            raise ValueError("bound arrays must be finite")
        if np.any(lo > hi):
            i, t = np.unravel_index(int(np.argmax(lo - hi)), lo.shape)
            raise ValueError(f"lo > hi at cell ({i}, {t}): {lo[i, t]} > {hi[i, t]}")
        self.lo = lo
        self.hi = hi
        self._uniform = None

    @classmethod
    def uniform(cls, n_rows: int, n_cols: int, lo: float, hi: float) -> "CellBounds":
        b = cls(np.full((n_rows, n_cols), float(lo)), np.full((n_rows, n_cols), float(hi)))
        b._uniform = (float(lo), float(hi))
        return b

    @property
    def n_rows(self) -> int:
        return self.lo.shape[0]

    @property
    def n_cols(self) -> int:
        return self.lo.shape[1]

    def widths(self, i: int) -> np.ndarray:
        return self.hi[i] - self.lo[i]

    def uniform_values(self):
        """(lo, hi) when every cell shares one interval, else None (the kernel then skips the arrays)."""
        if self._uniform is None and self.lo.size:
            lo0, hi0 = float(self.lo.flat[0]), float(self.hi.flat[0])
            if np.all(self.lo == lo0) and np.all(self.hi == hi0):
                self._uniform = (lo0, hi0)
            else:
                self._uniform = False
        return self._uniform or None
