"""Static reveal strategies (colbandit/baselines.py) on the device.

``full_rerank`` reveals every cell; ``doc_uniform`` / ``doc_top_margin`` buy
a fixed ``B = ceil(gamma * T)`` cells per row (baselines.py:49-86). All three
rank rows by the exactly rounded sum of the cells they revealed, ties to the
lower index (``_ranked_by_partial_sum``, baselines.py:38-41), and return the
reference's RunResult with the reveal trace in the reference's order.

The cells come from the float64 cell kernel (bit-equal to the reference for
16-bit inputs); the per-row exact partial sums are ``cbx_row_partial_fsum``
and the ranking is the device Top-K. Which cells a budgeted row buys is
decided on the host exactly as the reference decides it: numpy's
``Generator.choice(T, B, replace=False)`` per row in row order for
Doc-Uniform (a third-party algorithm the survey pins to numpy), the B widest
bounds with ties to the lower column for Doc-TopMargin.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .bandit import RunResult, ceil_cells
from .bounds import CellBounds

__all__ = ["BudgetConfig", "doc_uniform", "doc_top_margin", "full_rerank"]


@dataclass(frozen=True)
class BudgetConfig:
    """baselines.py:24-35 — per-row budget as a coverage fraction; B = ceil(gamma * T) cells."""

    gamma: float
    seed: int | tuple[int, ...] | None = 0

    def __post_init__(self) -> None:
        if not 0.0 < self.gamma <= 1.0:
            raise ValueError(f"gamma must be in (0, 1], got {self.gamma}")

    def cells_per_row(self, n_cols: int) -> int:
        return ceil_cells(self.gamma, n_cols)


def _check_k(k: int, n_rows: int) -> None:
    if not 0 <= k <= n_rows:
        raise ValueError(f"k must be in [0, {n_rows}], got {k}")


def _rank_rows(oracle, cols: np.ndarray, k: int) -> list[int]:
    """Device: exact partial sums of each row's chosen cells, then Top-K by (-sum, row)."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    from .batch import topk

    n_rows, b = cols.shape
    cells = oracle._device_cells()
    dev = cells.device
    cols_t = torch.from_numpy(np.ascontiguousarray(cols, dtype=np.int32)).to(dev)
    sums = torch.empty(n_rows, dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(lib.cbx_row_partial_fsum(cells.data_ptr(), int(cells.stride(0)), cols_t.data_ptr(), n_rows, b,
                                        sums.data_ptr(), status.data_ptr(), stream), "row_partial_fsum")
    if k == 0:
        return []
    if k <= 8192:
        off = torch.tensor([0, n_rows], dtype=torch.int64, device=dev)
        idx, _ = topk(sums, off, k, n_rows)
        order = idx[0].cpu().numpy()
    else:
        order = torch.argsort(-sums, stable=True)[:k].cpu().numpy()
    if int(status.item()):
        raise RuntimeError("exact partial-sum capacity exceeded")
    return [int(i) for i in order]


def _budget_result(oracle, cols: np.ndarray, k: int) -> RunResult:
    n_rows, n_cols = oracle.n_docs, oracle.n_query_tokens
    order = _rank_rows(oracle, cols, k)
    host = oracle._exact() if oracle._batch is not None else oracle._matrix
    rows = np.repeat(np.arange(n_rows), cols.shape[1])
    flat = cols.ravel()
    vals = host[rows, flat]
    trace = list(zip(rows.tolist(), flat.tolist(), vals.tolist()))
    oracle._reveal_count += len(trace)
    return RunResult(order, len(trace) / (n_rows * n_cols), trace, 0, "budget")


def doc_uniform(oracle, k: int, gamma: float, seed: int | tuple[int, ...] | None = 0) -> RunResult:
    """baselines.py:49-66 — B uniformly random cells per row, ranked by the partial sums."""
    budget = BudgetConfig(gamma, seed)
    n_rows, n_cols = oracle.n_docs, oracle.n_query_tokens
    _check_k(k, n_rows)
    b = budget.cells_per_row(n_cols)
    rng = np.random.default_rng(seed)
    cols = np.empty((n_rows, b), dtype=np.int32)
    for i in range(n_rows):
        cols[i] = rng.choice(n_cols, size=b, replace=False)
    return _budget_result(oracle, cols, k)


def doc_top_margin(oracle, bounds: CellBounds, k: int, gamma: float) -> RunResult:
    """baselines.py:69-86 — the B widest-bound cells per row (width ties to the lower column)."""
    BudgetConfig(gamma)
    n_rows, n_cols = oracle.n_docs, oracle.n_query_tokens
    if (bounds.n_rows, bounds.n_cols) != (n_rows, n_cols):
        raise ValueError("bounds shape does not match the matrix shape")
    _check_k(k, n_rows)
    b = ceil_cells(gamma, n_cols)
    width = np.asarray(bounds.hi, dtype=np.float64) - np.asarray(bounds.lo, dtype=np.float64)
    order = np.argsort(-width, axis=1, kind="stable")  # == lexsort((cols, -width)) per row
    return _budget_result(oracle, np.ascontiguousarray(order[:, :b], dtype=np.int32), k)


def full_rerank(oracle, k: int) -> RunResult:
    """baselines.py:89-97 — reveal every cell (row-major), rank by the exact row sums."""
    n_rows, n_cols = oracle.n_docs, oracle.n_query_tokens
    _check_k(k, n_rows)
    cols = np.tile(np.arange(n_cols, dtype=np.int32), (n_rows, 1))
    res = _budget_result(oracle, cols, k)
    return RunResult(res.topk, 1.0, res.reveals, 0, "budget")
