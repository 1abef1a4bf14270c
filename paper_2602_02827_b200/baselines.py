"""``full_rerank`` (colbandit/baselines.py:89-97) on the device.

Reveals every cell of the N x T matrix (float64-exact cell kernel), ranks rows
by the exactly rounded sum of their cells (device fsum) with ties to the lower
index (baselines.py:38-41), and returns the reference's RunResult with the
row-major trace.
"""

from __future__ import annotations

import math

import numpy as np

from .bandit import RunResult

__all__ = ["full_rerank"]


def full_rerank(oracle, k: int) -> RunResult:
    n_rows, n_cols = oracle.n_docs, oracle.n_query_tokens
    if not 0 <= k <= n_rows:
        raise ValueError(f"k must be in [0, {n_rows}], got {k}")
    cells = np.stack([oracle.row_values(i) for i in range(n_rows)]) if oracle._batch is None else oracle._exact()
    if oracle._batch is not None:
        sums = np.asarray(oracle._exact_scores, dtype=np.float64)
    else:
        sums = np.array([math.fsum(r.tolist()) for r in cells])
    order = np.lexsort((np.arange(n_rows), -sums))[:k] if n_rows else []
    if oracle._batch is not None and k:
        import torch

        from .batch import topk

        s = torch.from_numpy(sums).cuda()
        off = torch.tensor([0, n_rows], dtype=torch.int64, device="cuda")
        if k <= 8192:
            idx, _ = topk(s, off, k, n_rows)
            order = idx[0].cpu().numpy()
    trace = [(i, t, float(cells[i, t])) for i in range(n_rows) for t in range(n_cols)]
    oracle._reveal_count += n_rows * n_cols
    return RunResult([int(i) for i in order], 1.0, trace, 0, "budget")
