"""B200-native MaxSim scorer and Col-Bandit reranker (arxiv 2602.02827), drop-in for ``colbandit``.

Public surface mirrors the reference package's hot-path entry points:

* ``Similarity``, ``QueryTokens``, ``DocTokens``, ``MaxSimOracle`` (oracle.py)
* ``BanditConfig``, ``RunResult``, ``run`` (bandit.py); ``full_rerank`` (baselines.py)
* ``RadiusConfig``, ``CellBounds`` (bounds.py)

plus batched device entry points (``TokenBatch``, ``rerank_topk``,
``maxsim_scores``, ``run_batch``). All arithmetic runs in libcbx.so
(sm_100a); there is no CPU fallback.
"""

__version__ = "0.1.0"

from .bandit import BanditConfig, BanditJob, RunResult, ceil_cells, run, run_batch, select_ambiguous  # noqa: F401
from .baselines import full_rerank  # noqa: F401
from .batch import TokenBatch, exact_cells, maxsim_scores, rerank_topk, topk  # noqa: F401
from .bounds import CellBounds, RadiusConfig, fp_correction  # noqa: F401
from .oracle import DocTokens, MaxSimOracle, QueryTokens, Similarity  # noqa: F401
