"""Exhaustive MaxSim scoring, restated on the CPU (test infrastructure only).

Follows the reference semantics:

* cell H[i, t] = max_j <e_ij, q_t> computed as ``doc @ query.T`` in float64,
  optionally floored at 0 — colbandit/oracle.py:57-67 (token_scores) and
  oracle.py:205-215 (row_values: column max, cached per row);
* score S_i = math.fsum(H[i, :]) (exactly rounded) — oracle.py:222-227;
* Top-K = ``np.lexsort((arange(N), -S))[:k]``, ties to the lower row index,
  k outside [0, N] is a ValueError — oracle.py:229-235;
* the float64 upcast of every input — validation.py:8-23 (check_token_matrix).
"""

from __future__ import annotations

import math
from typing import Sequence

import numpy as np


def row_values(doc64: np.ndarray, query64: np.ndarray, clamp_negative: bool = False) -> np.ndarray:
    """All Lq cells of one document: column max of the (L_d, Lq) dot matrix."""
    s = np.asarray(doc64, dtype=np.float64) @ np.asarray(query64, dtype=np.float64).T
    if clamp_negative:
        np.maximum(s, 0.0, out=s)
    return s.max(axis=0)


def cell_matrix(query64: np.ndarray, docs64: Sequence[np.ndarray], clamp_negative: bool = False) -> np.ndarray:
    """The full N x Lq interaction matrix H (float64)."""
    return np.stack([row_values(d, query64, clamp_negative) for d in docs64])


def scores_from_cells(cells: np.ndarray) -> np.ndarray:
    """Exactly rounded row sums (math.fsum per row)."""
    return np.array([math.fsum(row.tolist()) for row in np.asarray(cells)], dtype=np.float64)


def exact_topk(scores: np.ndarray, k: int) -> list[int]:
    n = len(scores)
    if not 0 <= k <= n:
        raise ValueError(f"k must be in [0, {n}], got {k}")
    order = np.lexsort((np.arange(n), -np.asarray(scores, dtype=np.float64)))
    return [int(i) for i in order[:k]]


def score_query(query64: np.ndarray, docs64: Sequence[np.ndarray], k: int,
                clamp_negative: bool = False) -> tuple[np.ndarray, list[int], np.ndarray]:
    """(scores, top-K, cells) for one query — the P1 reference output."""
    cells = cell_matrix(query64, docs64, clamp_negative)
    scores = scores_from_cells(cells)
    return scores, exact_topk(scores, k), cells
