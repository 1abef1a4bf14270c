"""Pin the CPU oracle against golden vectors produced by the unmodified reference.

These run on CPU only; they are what makes the oracle trustworthy enough to
judge the CUDA path with (tests/golden/make_golden.py wrote the fixtures).
"""

import json
import math
import os

import numpy as np
import pytest

from oracle import bandit_ref, maxsim_ref
from oracle.pcg64_ref import PCG64Ref
from paper_2602_02827_b200 import workloads as W

from conftest import GOLDEN


def _load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _seed(s):
    return tuple(s) if isinstance(s, list) else s


# ---------------------------------------------------------------- PCG64
def test_pcg64_restatement_matches_numpy_streams():
    for stream in _load_json("pcg64_streams.json"):
        g = PCG64Ref(int(stream["state"]), int(stream["inc"]), stream["has_uint32"], stream["uinteger"])
        for kind, n, expect in stream["ops"]:
            got = g.random() if kind == "r" else g.integers(n)
            assert got == expect


def test_pcg64_seeding_matches_fixture_state():
    for stream in _load_json("pcg64_streams.json"):
        st = np.random.default_rng(_seed(stream["seed"])).bit_generator.state
        assert str(st["state"]["state"]) == stream["state"]
        assert str(st["state"]["inc"]) == stream["inc"]


# ---------------------------------------------------------------- P1
def test_maxsim_oracle_matches_reference_cells_scores_topk():
    z = np.load(os.path.join(GOLDEN, "p1_small.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    for m in meta:
        p = f"c{m['case']}_"
        q64 = W.to_float64(z[p + "query"], m["dtype"])
        t64 = W.to_float64(z[p + "tokens"], m["dtype"])
        off = z[p + "offsets"]
        docs = [t64[off[i]:off[i + 1]] for i in range(len(off) - 1)]
        scores, topk, cells = maxsim_ref.score_query(q64, docs, m["k"], m["clamp"])
        # fp16/bf16 products are exact in float64: cells bit-equal
        if m["dtype"] != "f32":
            np.testing.assert_array_equal(cells, z[p + "cells"])
            np.testing.assert_array_equal(scores, z[p + "scores"])
        else:
            np.testing.assert_allclose(cells, z[p + "cells"], rtol=0, atol=1e-15)
            np.testing.assert_allclose(scores, z[p + "scores"], rtol=1e-14)
        assert topk == z[p + "topk"].tolist()


def test_exact_topk_rejects_bad_k_and_breaks_ties_low():
    s = np.array([2.0, 2.0, 1.0, 2.0])
    assert maxsim_ref.exact_topk(s, 3) == [0, 1, 3]
    assert maxsim_ref.exact_topk(s, 0) == []
    with pytest.raises(ValueError, match="k must be in"):
        maxsim_ref.exact_topk(s, 5)


# ---------------------------------------------------------------- P2
def _run_case(case, indexed=False):
    cfg = dict(case["cfg"])
    cfg["seed"] = _seed(cfg["seed"])
    k = cfg.pop("k")
    cells = np.array(case["cells"], dtype=np.float64)
    if case["source"] == "matrix":
        lo, hi = np.array(case["lo"]), np.array(case["hi"])
    else:
        lo, hi = case["lo"], case["hi"]
    return bandit_ref.run(cells, lo, hi, k, indexed=indexed, **cfg)


@pytest.mark.parametrize("indexed", [False, True])
def test_bandit_oracle_matches_reference_trace_for_trace(indexed):
    # indexed: the sorted-key-list + lazy-heap ranking (the reference's structures) instead of a full sort
    for case in _load_json("p2_small.json"):
        res = _run_case(case, indexed)
        exp = case["result"]
        assert [list(r) for r in res.reveals] == exp["reveals"]
        assert res.topk == exp["topk"]
        assert res.iterations == exp["iterations"]
        assert res.terminated_by == exp["terminated_by"]
        assert res.coverage == exp["coverage"]


def test_token_cases_cells_match_reference():
    for case in _load_json("p2_small.json"):
        if case["source"] != "tokens":
            continue
        dt, d = case["dtype"], case["dim"]
        store = {"f32": np.float32, "f16": np.float16, "bf16": np.uint16}[dt]
        q = np.frombuffer(bytes.fromhex(case["query_hex"]), dtype=store).reshape(-1, d)
        toks = np.frombuffer(bytes.fromhex(case["tokens_hex"]), dtype=store).reshape(-1, d)
        off = case["offsets"]
        q64, t64 = W.to_float64(q, dt), W.to_float64(toks, dt)
        cells = maxsim_ref.cell_matrix(q64, [t64[off[i]:off[i + 1]] for i in range(len(off) - 1)],
                                       case["clamp"])
        exp = np.array(case["cells"])
        if dt == "f32":
            np.testing.assert_allclose(cells, exp, rtol=0, atol=1e-15)
        else:
            np.testing.assert_array_equal(cells, exp)
        full = bandit_ref.full_rerank(cells, case["cfg"]["k"])
        assert full.topk == case["full_rerank"]["topk"]
        assert len(full.reveals) == case["full_rerank"]["n_reveals"]


def test_bandit_oracle_edge_cases():
    cells = np.array([[0.6, 0.4], [0.2, 0.1]])
    assert bandit_ref.run(cells, 0.0, 1.0, 0) == bandit_ref.RefResult([], 0.0, [], 0, "separation")
    everyone = bandit_ref.run(cells, 0.0, 1.0, 2)
    assert everyone.reveals == [] and everyone.iterations == 1
    with pytest.raises(ValueError, match="exceeds the number of documents"):
        bandit_ref.run(cells, 0.0, 1.0, 3)
    # hard bounds already separate: zero reveals
    lo = np.array([[1.0, 1.0], [0.0, 0.0]])
    hi = np.array([[1.5, 1.5], [0.75, 0.75]])
    r = bandit_ref.run(np.array([[1.2, 1.3], [0.5, 0.5]]), lo, hi, 1)
    assert r.topk == [0] and r.reveals == [] and r.iterations == 1


def test_bound_scalars_frozen_values():
    # reference tests/test_bounds.py:63-68, 100-107
    assert bandit_ref.fp_correction(1, 32) == 1.0
    assert bandit_ref.fp_correction(32, 32) == 0.0
    assert bandit_ref.fp_correction(8, 32) == 0.78125
    assert bandit_ref.fp_correction(17, 32) == 0.4963235294117647
    assert bandit_ref.log_term(100, 32, 0.01, 1.0, "per-document") == math.log(100 / 0.01)
    assert bandit_ref.log_term(1, 1, 0.9, 0.5, "per-document") == 0.0


# ---------------------------------------------------------------- full-shape configs
@pytest.mark.parametrize("name,q", [("cfg1", 0), ("cfg2", 0), ("cfg2", 1), ("cfg2", 2), ("cfg3", 0), ("cfg3", 1),
                                    ("cfg5", 0), ("cfg5", 1)])
def test_config_fixture_fingerprint_and_p1(name, q):
    path = os.path.join(GOLDEN, f"{name}_q{q}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{name} q{q} fixture not generated")
    import hashlib

    z = np.load(path)
    case = W.gen_query(name, q)
    h = hashlib.sha256()
    for a in (case.query, case.doc_tokens, case.doc_offsets):
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    assert h.hexdigest() == bytes(z["fingerprint"]).decode(), "workload generator drifted"
    if name in ("cfg1", "cfg2"):
        scores, topk, _ = maxsim_ref.score_query(case.query64(), case.docs64(), W.CONFIGS[name].k)
        rtol = 1e-14 if name == "cfg1" else 0.0
        np.testing.assert_allclose(scores, z["scores"], rtol=rtol, atol=0)
        assert topk == z["topk"].tolist()


@pytest.mark.parametrize("q", [1, 2])
def test_cfg2_bandit_oracle_matches_reference(q):
    """The oracle loop on more full-shape cfg2 queries (seed (0, q)) against the reference's traces."""
    path = os.path.join(GOLDEN, f"cfg2_q{q}.npz")
    if not os.path.exists(path):
        pytest.skip("fixture not generated")
    z = np.load(path)
    case = W.gen_query("cfg2", q)
    cells = maxsim_ref.cell_matrix(case.query64(), case.docs64())
    res = bandit_ref.run(cells, -1.0, 1.0, 10, seed=(0, q))
    assert res.topk == z["a0_topk"].tolist()
    np.testing.assert_array_equal(np.array([(i, t) for i, t, _ in res.reveals]), z["a0_trace_it"])
    np.testing.assert_array_equal([v for *_, v in res.reveals], z["a0_trace_v"])
    assert res.coverage == z["a0_stats"][0] and res.iterations == z["a0_stats"][1]


def test_cfg1_bandit_oracle_matches_reference():
    z = np.load(os.path.join(GOLDEN, "cfg1_q0.npz"))
    case = W.gen_query("cfg1", 0)
    cells = maxsim_ref.cell_matrix(case.query64(), case.docs64())
    res = bandit_ref.run(cells, -1.0, 1.0, 5, seed=(0, 0))
    assert res.topk == z["a0_topk"].tolist()
    np.testing.assert_array_equal(np.array([(i, t) for i, t, _ in res.reveals]), z["a0_trace_it"])
    np.testing.assert_allclose([v for *_, v in res.reveals], z["a0_trace_v"], rtol=0, atol=1e-15)
    assert res.coverage == z["a0_stats"][0] and res.iterations == z["a0_stats"][1]


# ---------------------------------------------------------------- static-budget baselines
def test_budget_baselines_restatement_matches_reference():
    from oracle import baselines_ref

    for c in _load_json("budget_small.json"):
        cells = np.array(c["cells64"])
        u = baselines_ref.doc_uniform(cells, c["k"], c["gamma"], seed=_seed(c["seed"]))
        m = baselines_ref.doc_top_margin(cells, np.array(c["lo"]), np.array(c["hi"]), c["k"], c["gamma"])
        for got, want in ((u, c["uniform"]), (m, c["margin"])):
            assert got.topk == want["topk"]
            assert got.coverage == want["coverage"]
            assert [list(x) for x in got.reveals] == want["reveals"]
            assert got.terminated_by == want["terminated_by"] == "budget"
