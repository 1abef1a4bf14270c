"""B200-native MaxSim scorer and Col-Bandit reranker (arxiv 2602.02827), drop-in for ``colbandit``.

Public surface mirrors the reference package's hot-path entry points:

* ``Similarity``, ``QueryTokens``, ``DocTokens``, ``MaxSimOracle`` (oracle.py)
* ``BanditConfig``, ``RunResult``, ``run`` (bandit.py)
* ``full_rerank``, ``doc_uniform``, ``doc_top_margin`` (baselines.py)
* ``io``: CBM1 / CBH1 / manifest formats with loaders straight into HBM
* ``EvalInstance``, ``sweep_alpha``, ``sweep_budgets``, metrics (evaluation.py; the sweep is one launch)
* ``RadiusConfig``, ``CellBounds`` (bounds.py)
* ``generate_candidates``, ``derive_bounds``, ``CandidateSet``, ... (pipeline.py: Stage 1 on the device)
* ``ColBanditReranker``, ``RerankOutcome`` (reranker.py: the estimator facade)

plus batched device entry points (``TokenBatch``, ``rerank_topk``,
``maxsim_scores``, ``run_batch``). All arithmetic runs in libcbx.so
(sm_100a); there is no CPU fallback.
"""

__version__ = "0.1.0"

from .bandit import BanditConfig, BanditJob, RunResult, ceil_cells, run, run_batch, select_ambiguous  # noqa: F401
from .baselines import BudgetConfig, doc_top_margin, doc_uniform, full_rerank  # noqa: F401
from .batch import TokenBatch, exact_cells, maxsim_scores, rerank_topk, topk  # noqa: F401
from .bounds import (CellBounds, DecisionState, RadiusConfig, RowStats, compute_decision_state,  # noqa: F401
                     decision_interval, effective_radius, empirical_std, estimated_score, fp_correction, hard_bounds,
                     score_proxy)
from .oracle import DocTokens, MaxSimOracle, ObservationLedger, QueryTokens, Similarity, reveal  # noqa: F401
from .pipeline import (CandidateSet, TokenNeighbor, TokenNeighborList, derive_bounds,  # noqa: F401
                       generate_candidates, load_candidates, save_candidates)
from .reranker import ColBanditReranker, RerankOutcome  # noqa: F401
