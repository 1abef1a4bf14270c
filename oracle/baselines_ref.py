"""Static-budget baselines restated on the CPU (test infrastructure only).

colbandit/baselines.py:24-97: ``B = ceil_cells(gamma, T)`` cells per row;
Doc-Uniform draws them with ``np.random.default_rng(seed).choice(T, B,
replace=False)`` row by row (baselines.py:60-64), Doc-TopMargin takes the B
widest ``hi - lo`` columns with ties to the lower column (baselines.py:80-84);
rows are ranked by ``math.fsum`` of the revealed values, ties to the lower row
(baselines.py:38-41); coverage = reveals / (N T). Cells are the float64 N x T
matrix the reference's oracle would reveal.
"""

from __future__ import annotations

import math

import numpy as np

from .bandit_ref import RefResult, ceil_cells


def _check(gamma: float, k: int, n_rows: int) -> None:
    if not 0.0 < gamma <= 1.0:
        raise ValueError(f"gamma must be in (0, 1], got {gamma}")
    if not 0 <= k <= n_rows:
        raise ValueError(f"k must be in [0, {n_rows}], got {k}")


def _result(cells, picks, k):
    n_rows, n_cols = cells.shape
    trace = [(i, int(t), float(cells[i, t])) for i in range(n_rows) for t in picks[i]]
    sums = [math.fsum(float(cells[i, t]) for t in picks[i]) for i in range(n_rows)]
    order = sorted(range(n_rows), key=lambda i: (-sums[i], i))[:k]
    return RefResult(order, len(trace) / (n_rows * n_cols), trace, 0, "budget")


def doc_uniform(cells, k: int, gamma: float, seed=0) -> RefResult:
    cells = np.asarray(cells, dtype=np.float64)
    n_rows, n_cols = cells.shape
    _check(gamma, k, n_rows)
    b = ceil_cells(gamma, n_cols)
    rng = np.random.default_rng(seed)
    picks = [[int(t) for t in rng.choice(n_cols, size=b, replace=False)] for _ in range(n_rows)]
    return _result(cells, picks, k)


def doc_top_margin(cells, lo, hi, k: int, gamma: float) -> RefResult:
    cells = np.asarray(cells, dtype=np.float64)
    n_rows, n_cols = cells.shape
    _check(gamma, k, n_rows)
    b = ceil_cells(gamma, n_cols)
    width = np.broadcast_to(np.asarray(hi, np.float64) - np.asarray(lo, np.float64), cells.shape)
    cols = np.arange(n_cols)
    picks = [np.lexsort((cols, -width[i]))[:b].tolist() for i in range(n_rows)]
    return _result(cells, picks, k)
