"""Stage-1 candidate generation + ANN-derived bounds, restated on the CPU (test infrastructure only).

Citations are to /root/reference/pkg/src/colbandit:

* ``generate_candidates`` — pipeline.py:105-158: score every corpus token
  against every query token (the oracle's ``token_scores``, float64 GEMM,
  optional floor at 0 — oracle.py:57-67); per query token keep the top
  ``k_prime`` corpus tokens ranked by (-similarity, global token index)
  (``np.lexsort((arange, -scores))``, pipeline.py:137); candidates are the
  owners of kept tokens in corpus order; ``exact_cells[(row, t)]`` is the
  document's exact column max for every surfaced (doc, token) pair.
* ``derive_bounds`` — pipeline.py:161-185: lo = similarity floor; hi = the
  k'-th neighbour similarity of the token, overwritten by the exact column max
  for surfaced pairs; hi = max(hi, lo).
* ``rerank`` — reranker.py:106-149: Stage 1, pool oracle, ann/generic bounds,
  ``k = min(k, pool)``, seed ``(random_state, query_index)``, bandit run.

Output is plain arrays instead of the reference's dataclasses:
``neighbors`` is a list (per query token) of (doc_index, token_index,
similarity) tuples in rank order.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from . import bandit_ref, maxsim_ref


def token_scores(doc64: np.ndarray, query64: np.ndarray, clamp_negative: bool) -> np.ndarray:
    s = np.asarray(doc64, np.float64) @ np.asarray(query64, np.float64).T
    if clamp_negative:
        np.maximum(s, 0.0, out=s)
    return s


def generate_candidates(query64: np.ndarray, docs64: Sequence[np.ndarray], k_prime: int,
                        clamp_negative: bool = False):
    """Returns (doc_indices, exact_cells {(row, t): value}, neighbors per token)."""
    if len(docs64) == 0:
        raise ValueError("corpus must contain at least one document")
    if k_prime < 1:
        raise ValueError(f"k_prime must be at least 1, got {k_prime}")
    blocks = [token_scores(d, query64, clamp_negative) for d in docs64]
    row_max = [b.max(axis=0) for b in blocks]
    owner_doc = np.concatenate([np.full(b.shape[0], i, np.int64) for i, b in enumerate(blocks)])
    owner_tok = np.concatenate([np.arange(b.shape[0], dtype=np.int64) for b in blocks])
    allsc = np.concatenate(blocks, axis=0)
    total = allsc.shape[0]
    keep = min(k_prime, total)
    tiebreak = np.arange(total)
    neighbors, hit_docs, hit_pairs = [], set(), set()
    for t in range(query64.shape[0]):
        order = np.lexsort((tiebreak, -allsc[:, t]))[:keep]
        nbs = []
        for g in order:
            di = int(owner_doc[g])
            nbs.append((di, int(owner_tok[g]), float(allsc[g, t])))
            hit_docs.add(di)
            hit_pairs.add((di, t))
        neighbors.append(nbs)
    kept = sorted(hit_docs)
    row_of = {di: r for r, di in enumerate(kept)}
    exact = {(row_of[di], t): float(row_max[di][t]) for di, t in sorted(hit_pairs)}
    return kept, exact, neighbors


def derive_bounds(n_cand: int, exact: dict, neighbors, range_lo: float):
    n_tokens = len(neighbors)
    if n_cand == 0 or n_tokens == 0:
        raise ValueError("need at least one candidate and one query token")
    lo = np.full((n_cand, n_tokens), range_lo, dtype=np.float64)
    hi = np.empty((n_cand, n_tokens), dtype=np.float64)
    for t, nbs in enumerate(neighbors):
        hi[:, t] = nbs[-1][2]
    for (r, t), h in exact.items():
        hi[r, t] = h
    np.maximum(hi, lo, out=hi)
    return lo, hi


def rerank(query64: np.ndarray, docs64: Sequence[np.ndarray], *, k: int = 10, k_prime: int = 10,
           clamp_negative: bool = True, range_lo: float = -1.0, range_hi: float = 1.0,
           bounds_mode: str = "ann", random_state=0, query_index: int = 0, **bandit_kw):
    """One ``ColBanditReranker.rerank`` (reranker.py:106-149) for dot/cosine similarity with a
    fixed value range; returns (doc_indices of the Top-K, RefResult, candidate doc indices)."""
    lo_v = 0.0 if clamp_negative else range_lo
    kept, exact, neighbors = generate_candidates(query64, docs64, k_prime, clamp_negative)
    pool = [docs64[i] for i in kept]
    cells = maxsim_ref.cell_matrix(query64, pool, clamp_negative)
    if bounds_mode == "ann":
        lo, hi = derive_bounds(len(kept), exact, neighbors, lo_v)
    else:
        lo = np.full(cells.shape, lo_v)
        hi = np.full(cells.shape, range_hi)
    seed = None if random_state is None else (random_state, query_index)
    res = bandit_ref.run(cells, lo, hi, min(k, len(pool)), seed=seed, **bandit_kw)
    return [kept[i] for i in res.topk], res, kept
