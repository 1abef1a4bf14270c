"""Host-side Stage-1 / facade logic (no GPU): estimator params, ANN bound derivation, artifact I/O."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN


def test_reranker_params_match_reference_defaults():
    from sklearn.base import clone

    from paper_2602_02827_b200.reranker import ColBanditReranker

    est = ColBanditReranker()
    assert est.get_params() == {
        "k": 10, "k_prime": 10, "delta": 0.01, "alpha_ef": 1.0, "epsilon": 0.1,
        "explore_mode": "epsilon-greedy", "gamma_init": 0.0, "c": 1.0, "union_mode": "per-document",
        "similarity": "cosine", "clamp_negative": True, "bounds_mode": "ann", "random_state": 0,
    }
    c = clone(est.set_params(k=3, bounds_mode="generic"))
    assert c.get_params()["k"] == 3 and c.get_params()["bounds_mode"] == "generic"
    assert est._seed_for(4) == (0, 4)
    assert ColBanditReranker(random_state=None)._seed_for(4) is None


def _golden_candidates(ci):
    from paper_2602_02827_b200.pipeline import CandidateSet, TokenNeighbor, TokenNeighborList

    z = np.load(os.path.join(GOLDEN, "stage1_small.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    m = meta["cases"][ci]
    p = f"c{ci}_"
    cand_idx = z[p + "cand"].tolist()
    exact = {(int(r), int(t)): float(v) for (r, t), v in zip(z[p + "exact_rt"], z[p + "exact_v"])}
    cand = CandidateSet(tuple(f"d{i:03d}" for i in cand_idx), tuple(cand_idx), exact)
    nls = [TokenNeighborList(t, tuple(TokenNeighbor(f"d{d:03d}", int(d), int(j), float(s))
                                      for d, j, s in zip(z[p + "nb_doc"][t], z[p + "nb_tok"][t], z[p + "nb_sim"][t])))
           for t in range(z[p + "nb_doc"].shape[0])]
    return m, z, p, cand, nls


@pytest.mark.parametrize("ci", range(6))
def test_derive_bounds_matches_reference(ci):
    from paper_2602_02827_b200.oracle import Similarity
    from paper_2602_02827_b200.pipeline import derive_bounds

    m, z, p, cand, nls = _golden_candidates(ci)
    sim = Similarity(kind="dot", clamp_negative=m["clamp"])
    b = derive_bounds(cand, nls, sim)
    np.testing.assert_array_equal(b.hi, z[p + "hi"])
    np.testing.assert_array_equal(b.lo, z[p + "lo"])


def test_candidate_artifact_round_trip(tmp_path):
    from paper_2602_02827_b200.oracle import Similarity
    from paper_2602_02827_b200.pipeline import (CandidateSet, TokenNeighbor, TokenNeighborList, derive_bounds,
                                                load_candidates, save_candidates)

    m, z, p, cand, nls = _golden_candidates(1)
    sim = Similarity(kind="dot", clamp_negative=m["clamp"])
    b = derive_bounds(cand, nls, sim)
    path = tmp_path / "cand.json"
    save_candidates(path, cand, nls, b, k_prime=m["k_prime"], similarity=sim, query_path="q.npy")
    got = load_candidates(path)
    assert got["doc_indices"] == list(cand.doc_indices)
    assert got["kth_sim"] == [nl.kth_similarity for nl in nls]
    np.testing.assert_array_equal(np.array(got["hi"]), b.hi)
    assert got["similarity"]["clamp_negative"] is True and got["query_path"] == "q.npy"
    (tmp_path / "bad.json").write_text(json.dumps({"format": "x"}))
    with pytest.raises(ValueError, match="not a candidate artifact"):
        load_candidates(tmp_path / "bad.json")
    with pytest.raises(ValueError, match="non-increasing"):
        TokenNeighborList(0, (TokenNeighbor("a", 0, 0, 0.1), TokenNeighbor("b", 1, 0, 0.2)))
    with pytest.raises(ValueError, match="distinct"):
        CandidateSet(("a", "a"), (0, 1), {})
