"""Host-side interval scalars and ledger helpers (bounds.py / bandit.py mirrors), no GPU."""

import math

import numpy as np
import pytest

from oracle import bandit_ref
from paper_2602_02827_b200 import bandit as B
from paper_2602_02827_b200 import bounds as BD
from paper_2602_02827_b200.oracle import ObservationLedger, reveal


class _M:
    def __init__(self, m):
        self.m = np.asarray(m, dtype=np.float64)
        self.n_docs, self.n_query_tokens = self.m.shape

    def _charge(self, i, t):
        return float(self.m[i, t])


def test_scalars_match_the_pinned_oracle():
    for T in (1, 2, 7, 32, 64):
        for n in range(1, T + 1):
            assert BD.fp_correction(n, T) == bandit_ref.fp_correction(n, T)
    assert BD.fp_correction(1, 9) == 1.0 and BD.fp_correction(9, 9) == 0.0
    with pytest.raises(ValueError, match="fp_correction needs"):
        BD.fp_correction(0, 4)
    cfg = BD.RadiusConfig(alpha_ef=0.3, delta=0.05, c=2.0, union_mode="per-document-and-size")
    assert cfg.log_term(100, 32) == bandit_ref.log_term(100, 32, 0.05, 2.0, "per-document-and-size")
    assert BD.RadiusConfig(delta=0.5, c=0.1).log_term(1, 1) == 0.0  # clamped at zero


def test_row_stats_radius_and_interval():
    s = BD.RowStats.from_values([0.5, 0.25, 0.75])
    assert (s.n, s.total, s.mean) == (3, 1.5, 0.5) and math.isclose(s.m2, 0.125)
    assert BD.empirical_std(s) == math.sqrt(0.125 / 2)
    assert BD.estimated_score(s, 6) == 3.0 and BD.estimated_score(s, 3) == 1.5
    with pytest.raises(ValueError, match="undefined for n=1"):
        BD.empirical_std(BD.RowStats.from_values([1.0]))
    with pytest.raises(ValueError, match="unobserved row"):
        BD.estimated_score(BD.RowStats.from_values([]), 4)
    cfg = BD.RadiusConfig()
    assert BD.effective_radius(BD.RowStats.from_values([1.0]), 4, cfg, 10) == math.inf
    assert BD.effective_radius(BD.RowStats.from_values([1.0, 0.5, 0.25, 0.0]), 4, cfg, 10) == 0.0  # full reveal
    assert BD.decision_interval(None, 1.0, -2.0, 3.0) == (-2.0, 3.0)
    assert BD.decision_interval(1.0, math.inf, -2.0, 3.0) == (-2.0, 3.0)
    assert BD.decision_interval(1.0, 0.5, -2.0, 3.0) == (0.5, 1.5)
    assert BD.decision_interval(5.0, 0.5, -2.0, 3.0) == (3.0, 3.0)  # estimate above the envelope: both clipped


def test_decision_state_over_a_ledger():
    m = [[0.5, 0.25, 1.0, -0.5], [0.125, 0.0, -0.25, 0.75]]
    o = _M(m)
    bnd = BD.CellBounds.uniform(2, 4, -1.0, 1.0)
    led = ObservationLedger(2, 4)
    st0 = BD.compute_decision_state(led, bnd, 0, BD.RadiusConfig())
    assert st0.est_score is None and (st0.hard_lo, st0.hard_hi) == (-4.0, 4.0) and BD.score_proxy(st0) == 0.0
    for t in (2, 0):
        reveal(led, o, 0, t)
    st = BD.compute_decision_state(led, bnd, 0, BD.RadiusConfig())
    assert (st.hard_lo, st.hard_hi) == (-0.5, 3.5) and st.est_score == 3.0 and BD.score_proxy(st) == 3.0
    assert st.lcb <= st.ucb and st.width == st.ucb - st.lcb
    for t in (1, 3):
        reveal(led, o, 0, t)
    full = BD.compute_decision_state(led, bnd, 0, BD.RadiusConfig())
    assert full.hard_lo == full.hard_hi == math.fsum(m[0]) == full.lcb == full.ucb


def test_ledger_driven_helpers():
    o = _M(np.arange(12, dtype=np.float64).reshape(3, 4) / 16)
    led = ObservationLedger(3, 4)
    B.init_one_per_row(o, led, np.random.default_rng(3))
    assert [led.row_count(i) for i in range(3)] == [1, 1, 1]
    r = np.random.default_rng(3)
    assert [t for _, t, _ in led.trace] == [int(r.integers(4)) for _ in range(3)]
    bnd = BD.CellBounds(np.zeros((3, 4)), np.array([[1, 3, 3, 2]] * 3, dtype=np.float64))
    t = B.select_token(led, bnd, 0, 0.0, np.random.default_rng(0))
    assert t == min(c for c in led.unobserved_cols(0) if bnd.hi[0, c] == max(bnd.hi[0, led.unobserved_cols(0)]))
    led2 = ObservationLedger(3, 4)
    B.static_warmup(o, led2, 0.5, np.random.default_rng(9))
    assert led2.observed_count == 6
    with pytest.raises(ValueError, match="gamma_init"):
        B.static_warmup(o, led2, 1.5, np.random.default_rng(9))
    full = ObservationLedger(1, 2)
    o1 = _M([[0.0, 1.0]])
    reveal(full, o1, 0, 0)
    reveal(full, o1, 0, 1)
    with pytest.raises(ValueError, match="fully revealed"):
        B.select_token(full, BD.CellBounds.uniform(1, 2, 0, 1), 0, 0.5, np.random.default_rng(0))
