"""Drop-in ``ColBanditReranker`` (colbandit/reranker.py) over the B200 kernels.

Same constructor parameters, defaults, fitted attributes, validation
messages and outputs as reranker.py:41-163. ``fit`` uploads the corpus to
HBM once (``batch.Corpus``); ``rerank`` runs Stage 1 on the device
(pipeline.stage1: tcgen05 scan + float64 refine), gathers the candidate pool
from the resident corpus, derives the ANN (or generic) bounds and runs the
Col-Bandit loop in the device kernel with the seed ``(random_state,
query_index)``. ``predict`` answers a whole batch with one Stage-1 scan and
one bandit launch (one CTA per query) instead of a per-query loop; results
are identical to calling ``rerank`` per query.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .bandit import BanditConfig, BanditJob, RunResult, run_batch
from .bounds import CellBounds
from .oracle import DocTokens, QueryTokens, Similarity
from .pipeline import CandidateSet, derive_bounds, stage1
from .validation import check_unit_norm

try:  # the reference's facade is a scikit-learn estimator (get_params / set_params / clone)
    from sklearn.base import BaseEstimator
except ImportError:  # pragma: no cover
    BaseEstimator = object

__all__ = ["RerankOutcome", "ColBanditReranker"]


@dataclass(frozen=True)
class RerankOutcome:
    """reranker.py:25-38."""

    doc_ids: tuple[str, ...]
    doc_indices: tuple[int, ...]
    coverage: float
    reveals: int
    candidates: CandidateSet
    result: RunResult


class ColBanditReranker(BaseEstimator):
    """Adaptive Top-K reranker over token-level interactions (reranker.py:41-163)."""

    def __init__(
        self,
        k: int = 10,
        k_prime: int = 10,
        delta: float = 0.01,
        alpha_ef: float = 1.0,
        epsilon: float = 0.1,
        explore_mode: str = "epsilon-greedy",
        gamma_init: float = 0.0,
        c: float = 1.0,
        union_mode: str = "per-document",
        similarity: str = "cosine",
        clamp_negative: bool = True,
        bounds_mode: str = "ann",
        random_state: int = 0,
    ):
        self.k = k
        self.k_prime = k_prime
        self.delta = delta
        self.alpha_ef = alpha_ef
        self.epsilon = epsilon
        self.explore_mode = explore_mode
        self.gamma_init = gamma_init
        self.c = c
        self.union_mode = union_mode
        self.similarity = similarity
        self.clamp_negative = clamp_negative
        self.bounds_mode = bounds_mode
        self.random_state = random_state

    # ------------------------------------------------------------------ fit
    def fit(self, X, y=None):
        """Store the corpus (a list of DocTokens or of (count, dim) arrays) in device memory.

        A ``batch.Corpus`` (already HBM-resident, e.g. built from one token tensor + offsets) is adopted
        as is, without a host round trip.
        """
        from .batch import Corpus

        if isinstance(X, Corpus):
            if self.bounds_mode not in ("ann", "generic"):
                raise ValueError(f"bounds_mode must be 'ann' or 'generic', got {self.bounds_mode!r}")
            if X.doc_ids is None:
                X.doc_ids = [f"doc{i:04d}" for i in range(X.n_docs)]
            self.docs_ = X
            self.dim_ = X.dim
            self.similarity_ = Similarity(kind=self.similarity, clamp_negative=self.clamp_negative)
            self.corpus_ = X
            return self
        if not X:
            raise ValueError("corpus must contain at least one document")
        docs = []
        for i, item in enumerate(X):
            if isinstance(item, DocTokens):
                docs.append(item)
            else:
                docs.append(DocTokens(f"doc{i:04d}", item if _is_tensor(item) else np.asarray(item)))
        dims = {d.vectors.shape[1] for d in docs}
        if len(dims) != 1:
            raise ValueError(f"documents disagree on embedding dim: {sorted(dims)}")
        if self.bounds_mode not in ("ann", "generic"):
            raise ValueError(f"bounds_mode must be 'ann' or 'generic', got {self.bounds_mode!r}")
        self.docs_ = docs
        self.dim_ = dims.pop()
        self.similarity_ = Similarity(kind=self.similarity, clamp_negative=self.clamp_negative)
        self.corpus_ = Corpus.from_docs(docs, clamp_negative=self.clamp_negative)
        return self

    # ------------------------------------------------------------------ answer
    def rerank(self, query, query_index: int = 0) -> RerankOutcome:
        """Answer one query (a QueryTokens or a (T, dim) array) in detail."""
        return self._answer([query], [query_index])[0]

    def predict(self, X) -> list[tuple[str, ...]]:
        """Top-K doc_ids, best-first, for each query in X (one batched device pass)."""
        self._check_fitted()
        X = list(X)
        return [o.doc_ids for o in self._answer(X, list(range(len(X))))]

    def rerank_batch(self, queries, query_indices=None) -> list[RerankOutcome]:
        """``rerank`` for many queries at once (one Stage-1 scan, one bandit launch)."""
        queries = list(queries)
        idx = list(range(len(queries))) if query_indices is None else list(query_indices)
        return self._answer(queries, idx)

    def _answer(self, queries, indices) -> list[RerankOutcome]:
        self._check_fitted()
        qs = []
        for q in queries:
            if not isinstance(q, QueryTokens):
                q = QueryTokens(q if _is_tensor(q) else np.asarray(q))
            if q.vectors.shape[1] != self.dim_:
                raise ValueError(f"query dim {q.vectors.shape[1]} does not match corpus dim {self.dim_}")
            qs.append(q)
        if not qs:
            return []
        results, pool_batch = stage1(self.corpus_, qs, self.k_prime, self.similarity_.clamp_negative)
        jobs = []
        for qi, (q, r) in enumerate(zip(qs, results)):
            cand = r.candidates
            if self.similarity_.kind == "cosine":  # MaxSimOracle construction (oracle.py:125-131)
                check_unit_norm(q.vectors, "query vectors")
                self._check_pool_norms(pool_batch, qi, cand)
            T = q.vectors.shape[0]
            if self.bounds_mode == "ann":
                bounds = derive_bounds(cand, r.neighbor_lists, self.similarity_)
            else:
                bounds = CellBounds.uniform(len(cand), T, self.similarity_.range_lo, self.similarity_.range_hi)
            cfg = BanditConfig(
                k=min(self.k, len(cand)),
                delta=self.delta,
                alpha_ef=self.alpha_ef,
                epsilon=self.epsilon,
                explore_mode=self.explore_mode,
                gamma_init=self.gamma_init,
                c=self.c,
                union_mode=self.union_mode,
                seed=self._seed_for(indices[qi]),
            )
            jobs.append(BanditJob(cfg, len(cand), T, qi, int(pool_batch.host_offsets[2][qi]), bounds))
        runs = run_batch(jobs, batch=pool_batch)
        out = []
        for r, res in zip(results, runs):
            cand = r.candidates
            out.append(RerankOutcome(
                doc_ids=tuple(cand.doc_ids[i] for i in res.topk),
                doc_indices=tuple(cand.doc_indices[i] for i in res.topk),
                coverage=res.coverage,
                reveals=len(res.reveals),
                candidates=cand,
                result=res,
            ))
        return out

    def _check_pool_norms(self, pool_batch, qi, cand) -> None:
        qd = pool_batch.host_offsets[2]
        do = pool_batch.host_offsets[1]
        a, b = int(do[qd[qi]]), int(do[qd[qi + 1]])
        rows = pool_batch.d_tokens[a:b].double().cpu().numpy()
        starts = do[qd[qi]:qd[qi + 1] + 1] - a
        for j, di in enumerate(cand.doc_indices):
            check_unit_norm(rows[starts[j]:starts[j + 1]], f"doc {cand.doc_ids[j]!r} vectors")

    def _seed_for(self, query_index: int):
        if self.random_state is None:
            return None
        return (self.random_state, query_index)

    def _check_fitted(self) -> None:
        if not hasattr(self, "docs_"):
            raise RuntimeError("this reranker is not fitted yet; call fit(corpus) first")


def _is_tensor(x) -> bool:
    try:
        import torch

        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False
