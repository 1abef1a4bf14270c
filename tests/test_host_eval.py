"""Evaluation metrics and frontier bookkeeping (host logic, no GPU)."""

import math

import pytest

from paper_2602_02827_b200 import evaluation as E


def test_metrics_known_values():
    assert E.overlap_at_k([1, 2, 3], [3, 4, 1], 3) == 2 / 3
    with pytest.raises(ValueError, match="exactly k=3"):
        E.overlap_at_k([1, 2], [1, 2, 3], 3)
    assert E.recall_at_k(["a", "b", "c"], {"c", "z"}, 2) == 0.0
    assert E.recall_at_k(["a", "b", "c"], {"c", "z"}, 3) == 0.5
    assert E.mrr_at_k(["a", "b", "c"], {"b"}, 3) == 0.5
    assert E.ndcg_at_k(["a", "b"], {"b"}, 2) == (1 / math.log2(3)) / 1.0
    with pytest.raises(ValueError, match="relevant set is empty"):
        E.mrr_at_k(["a"], set(), 1)
    with pytest.raises(ValueError, match="k must be at least 1"):
        E.ndcg_at_k(["a"], {"a"}, 0)


def test_seeds_grids_and_aggregation(tmp_path):
    assert E.instance_seed(None, 3) is None
    assert E.instance_seed(5, 3) == (5, 3)
    assert E.instance_seed((5, 1), 3) == (5, 1, 3)
    assert len(E.DEFAULT_ALPHA_GRID) == 16 and E.DEFAULT_ALPHA_GRID[0] == 1e-3 and E.DEFAULT_ALPHA_GRID[-1] == 1.0
    assert E.DEFAULT_GAMMA_GRID[0] == 0.05 and E.DEFAULT_GAMMA_GRID[-1] == 1.0
    p = E.aggregate_frontier("bandit", 0.1, [(0.5, 1.0, None, None, None), (0.25, 0.5, 1.0, 0.5, 1.0)])
    assert p.mean_coverage == 0.375 and p.overlap_at_k == 0.75 and p.recall_at_k == 1.0 and p.n_queries == 2
    assert p.row()[:2] == ["bandit", "0.1"]
    q = E.aggregate_frontier("bandit", 0.2, [(0.1, 0.5, None, None, None)])
    assert q.row()[5:8] == ["", "", ""]
    assert E.coverage_required([p, q], 0.7) is p and E.coverage_required([p, q], 0.9) is None
    qrels = tmp_path / "q.txt"
    qrels.write_text("q1 0 d1 1\nq1 0 d2 0\n\nq2 0 d3 -1\n")
    assert E.read_qrels(qrels) == {"q1": {"d1"}, "q2": set()}
    qrels.write_text("q1 0 d1\n")
    with pytest.raises(ValueError, match="expected 4 fields"):
        E.read_qrels(qrels)
