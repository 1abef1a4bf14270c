"""Pin the Stage-1 / facade CPU restatement against the reference's golden outputs (CPU only)."""

import json
import os

import numpy as np
import pytest

from oracle import stage1_ref
from paper_2602_02827_b200 import workloads as W

from conftest import GOLDEN


def _load():
    z = np.load(os.path.join(GOLDEN, "stage1_small.npz"))
    return z, json.loads(bytes(z["meta"]).decode())


def _case(z, m):
    p = f"c{m['case']}_"
    t64 = W.to_float64(z[p + "tokens"], m["dtype"])
    off = z[p + "offsets"]
    docs = [t64[off[i]:off[i + 1]] for i in range(len(off) - 1)]
    return W.to_float64(z[p + "query"], m["dtype"]), docs, p


def test_generate_candidates_restatement_matches_reference():
    z, meta = _load()
    for m in meta["cases"]:
        q64, docs, p = _case(z, m)
        kept, exact, nbs = stage1_ref.generate_candidates(q64, docs, m["k_prime"], m["clamp"])
        np.testing.assert_array_equal(kept, z[p + "cand"])
        np.testing.assert_array_equal([[n[0] for n in nl] for nl in nbs], z[p + "nb_doc"])
        np.testing.assert_array_equal([[n[1] for n in nl] for nl in nbs], z[p + "nb_tok"])
        np.testing.assert_array_equal([[n[2] for n in nl] for nl in nbs], z[p + "nb_sim"])
        got = sorted(exact.items())
        np.testing.assert_array_equal(np.array([k for k, _ in got]).reshape(-1, 2), z[p + "exact_rt"])
        np.testing.assert_array_equal([v for _, v in got], z[p + "exact_v"])
        lo, hi = stage1_ref.derive_bounds(len(kept), exact, nbs, 0.0 if m["clamp"] else -1.0)
        np.testing.assert_array_equal(hi, z[p + "hi"])
        np.testing.assert_array_equal(lo, z[p + "lo"])


def test_generate_candidates_errors():
    with pytest.raises(ValueError, match="at least one document"):
        stage1_ref.generate_candidates(np.ones((1, 2)), [], 3)
    with pytest.raises(ValueError, match="k_prime must be at least 1"):
        stage1_ref.generate_candidates(np.ones((1, 2)), [np.ones((1, 2))], 0)


@pytest.mark.parametrize("fi", range(5))
def test_facade_restatement_matches_reference(fi):
    z, meta = _load()
    f = meta["facade"][fi]
    m = meta["cases"][f["corpus_case"]]
    _, docs, _ = _case(z, m)
    for qi, want in enumerate(f["outcomes"]):
        q64 = W.to_float64(z[f"f{fi}_q{qi}"], m["dtype"])
        top, res, kept = stage1_ref.rerank(q64, docs, k=f["k"], k_prime=10, clamp_negative=f["clamp"],
                                           bounds_mode=f["bounds_mode"], random_state=f["random_state"],
                                           query_index=qi)
        assert kept == want["cand"]
        assert top == want["doc_indices"]
        assert [list(x) for x in res.reveals] == want["trace"]
        assert res.iterations == want["iterations"] and res.terminated_by == want["terminated_by"]
        assert [f"doc{i:04d}" for i in top] == f["predict"][qi]
