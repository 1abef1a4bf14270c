"""Bound configuration objects and interval scalars of the reference, mirrored for the drop-in API.

``RadiusConfig`` / ``CellBounds`` keep the reference's field names, defaults,
validation and messages (colbandit/bounds.py:112-191). The interval
arithmetic of the loop (hard bounds, radius, decision interval, score proxy —
bounds.py:72-263) runs inside the bandit kernel (csrc/bandit.cu
``row_interval``); the scalar functions below are the same arithmetic on the
host for callers that drive their own ledger (``oracle.ObservationLedger``).
``log_term`` is always evaluated here with ``math.log`` exactly as the
reference does (bounds.py:138-143), because a device ``log`` may differ in
the last ulp.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

UNION_MODES = ("per-document", "per-document-and-size")

__all__ = ["RadiusConfig", "CellBounds", "UNION_MODES", "fp_correction", "RowStats", "empirical_std",
           "estimated_score", "effective_radius", "hard_bounds", "decision_interval", "DecisionState",
           "compute_decision_state", "score_proxy"]


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


# ---------------------------------------------------------------- interval scalars (bounds.py:45-263)
@dataclass(frozen=True)
class RowStats:
    """Revealed-cell statistics of one row: count, exact (fsum) total, Welford mean and m2."""

    n: int
    total: float
    mean: float
    m2: float

    @classmethod
    def from_values(cls, values) -> "RowStats":
        """Two-pass construction (bounds.py:59-69)."""
        vals = [float(v) for v in values]
        n = len(vals)
        if n == 0:
            return cls(0, 0.0, 0.0, 0.0)
        total = math.fsum(vals)
        mean = total / n
        return cls(n, total, mean, math.fsum((v - mean) ** 2 for v in vals))


def empirical_std(stats: RowStats) -> float:
    """bounds.py:72-80 — unbiased sample std; undefined below two observations."""
    if stats.n <= 1:
        raise ValueError(f"empirical_std undefined for n={stats.n}; need at least 2 observations")
    return math.sqrt(max(stats.m2, 0.0) / (stats.n - 1))


def estimated_score(stats: RowStats, n_cols: int) -> float:
    """bounds.py:83-94 — T * (total / n); the exact total at full reveal."""
    if stats.n == 0:
        raise ValueError("estimated score undefined for an unobserved row")
    if stats.n == n_cols:
        return stats.total
    return n_cols * (stats.total / stats.n)


def effective_radius(stats: RowStats, n_cols: int, cfg: RadiusConfig, n_rows: int) -> float:
    """bounds.py:146-158 — alpha * T * sigma * sqrt(2 log_term / n) * sqrt(rho_n); inf for n <= 1."""
    if stats.n <= 1:
        return math.inf
    sigma = empirical_std(stats)
    rho = fp_correction(stats.n, n_cols)
    return cfg.alpha_ef * n_cols * sigma * math.sqrt(2.0 * cfg.log_term(n_rows, n_cols) / stats.n) * math.sqrt(rho)


def hard_bounds(ledger, bounds: CellBounds, i: int) -> tuple[float, float]:
    """bounds.py:194-208 — revealed values plus unrevealed support bounds, exactly rounded sums."""
    if (ledger.n_rows, ledger.n_cols) != (bounds.n_rows, bounds.n_cols):
        raise ValueError("ledger and bounds shapes differ")
    observed = math.fsum(ledger.row_values(i))
    rest = ledger.unobserved_cols(i)
    return (observed + math.fsum(float(bounds.lo[i, t]) for t in rest),
            observed + math.fsum(float(bounds.hi[i, t]) for t in rest))


def decision_interval(est_score, radius: float, hard_lo: float, hard_hi: float) -> tuple[float, float]:
    """bounds.py:211-225 — the statistical interval clipped into the hard envelope (both ends)."""
    if est_score is None or math.isinf(radius):
        return hard_lo, hard_hi
    return min(max(hard_lo, est_score - radius), hard_hi), max(min(hard_hi, est_score + radius), hard_lo)


@dataclass(frozen=True)
class DecisionState:
    """bounds.py:228-241."""

    est_score: float | None
    hard_lo: float
    hard_hi: float
    radius: float
    lcb: float
    ucb: float

    @property
    def width(self) -> float:
        return self.ucb - self.lcb


def compute_decision_state(ledger, bounds: CellBounds, i: int, radius_cfg: RadiusConfig) -> DecisionState:
    """bounds.py:244-256."""
    stats = ledger.row_stats(i)
    h_lo, h_hi = hard_bounds(ledger, bounds, i)
    est = None if stats.n == 0 else estimated_score(stats, ledger.n_cols)
    radius = effective_radius(stats, ledger.n_cols, radius_cfg, ledger.n_rows)
    lcb, ucb = decision_interval(est, radius, h_lo, h_hi)
    return DecisionState(est, h_lo, h_hi, radius, lcb, ucb)


def score_proxy(state: DecisionState) -> float:
    """bounds.py:259-263 — the estimate, or the hard midpoint before any reveal."""
    if state.est_score is None:
        return 0.5 * (state.hard_lo + state.hard_hi)
    return state.est_score
