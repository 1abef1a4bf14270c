"""Stage-1 scan, ANN bounds and the ColBanditReranker facade on the B200 against the reference goldens.

Everything here is integer / ordering work on exact float64 similarities
(16-bit inputs: exact products, exact sums), so the bar is bit-equality:
neighbour lists (doc, token, similarity, order), candidate sets, exact cells,
hi/lo bounds, and for the facade the full reveal trace of every query.
The tcgen05 scan (fp32 filter + float64 refine) must equal the float64 SIMT
scan bit for bit on every input, including duplicated tokens (ties) and
clamped zero ties (where it hands over to the SIMT scan).
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2602_02827_b200 import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _t(x, dt):
    from paper_2602_02827_b200.batch import to_torch_tokens

    return to_torch_tokens(x, "bf16" if dt == "bf16" else None)


def _load():
    z = np.load(os.path.join(GOLDEN, "stage1_small.npz"))
    return z, json.loads(bytes(z["meta"]).decode())


def _docs(z, m):
    from paper_2602_02827_b200.oracle import DocTokens

    p = f"c{m['case']}_"
    toks, off = z[p + "tokens"], z[p + "offsets"]
    t = _t(toks, m["dtype"])
    return [DocTokens(f"d{i:03d}", t[off[i]:off[i + 1]]) for i in range(len(off) - 1)], p


@pytest.mark.parametrize("path", ["auto", "simt", "tc"])
def test_generate_candidates_matches_reference_golden(path):
    from paper_2602_02827_b200.oracle import QueryTokens, Similarity
    from paper_2602_02827_b200.pipeline import derive_bounds, generate_candidates, stage1_topk

    z, meta = _load()
    ran_tc = 0
    for m in meta["cases"]:
        docs, p = _docs(z, m)
        n_tok = int(z[p + "offsets"][-1])
        if path == "tc" and (n_tok < 8192 or m["k_prime"] > 64):
            continue
        sim = Similarity(kind="dot", range_lo=-1.0, range_hi=1.0, clamp_negative=m["clamp"])
        q = QueryTokens(_t(z[p + "query"], m["dtype"]))
        cand, nls = generate_candidates(q, docs, sim, m["k_prime"], path=path)
        if "tc" in stage1_topk.last_paths:
            ran_tc += 1
        np.testing.assert_array_equal([[nb.doc_index for nb in nl.neighbors] for nl in nls], z[p + "nb_doc"])
        np.testing.assert_array_equal([[nb.token_index for nb in nl.neighbors] for nl in nls], z[p + "nb_tok"])
        np.testing.assert_array_equal([[nb.similarity for nb in nl.neighbors] for nl in nls], z[p + "nb_sim"])
        assert [nb.doc_id for nb in nls[0].neighbors] == [f"d{d:03d}" for d in z[p + "nb_doc"][0]]
        np.testing.assert_array_equal(cand.doc_indices, z[p + "cand"])
        got = sorted(cand.exact_cells.items())
        np.testing.assert_array_equal(np.array([k for k, _ in got]).reshape(-1, 2), z[p + "exact_rt"])
        np.testing.assert_array_equal([v for _, v in got], z[p + "exact_v"])
        bnd = derive_bounds(cand, nls, sim)
        np.testing.assert_array_equal(bnd.hi, z[p + "hi"])
        np.testing.assert_array_equal(bnd.lo, z[p + "lo"])
    if path == "tc":
        assert ran_tc >= 2


@pytest.mark.parametrize("dt,d,n_tok,rows,kp,clamp,dup", [
    ("f16", 128, 60_000, 32, 10, False, 0.0),
    ("bf16", 128, 50_000, 300, 10, True, 0.05),   # 3 row blocks
    ("f16", 256, 40_000, 64, 64, False, 0.0),
    ("bf16", 64, 30_000, 128, 1, True, 0.2),
    ("f16", 96, 20_000, 7, 33, False, 0.3),       # dim not a multiple of 64, heavy duplication
    ("bf16", 64, 700_000, 40, 10, True, 0.01),    # large enough for the threshold pre-pass
    ("f16", 128, 900_000, 200, 5, False, 0.0),    # pre-pass with two row blocks
    ("f16", 128, 60_000, 100, 128, False, 0.0),   # k' > 64: 128 sorted tops per row
    ("bf16", 128, 800_000, 40, 128, True, 0.02),  # k' = 128 with the pre-pass
    ("f16", 128, 120_000, 32, 256, False, 0.1),   # k' = 256 (64-row tiles)
    ("bf16", 256, 60_000, 16, 100, True, 0.0),    # d = 256, k' = 100
])
def test_tc_scan_equals_simt_scan(dt, d, n_tok, rows, kp, clamp, dup):
    from paper_2602_02827_b200.batch import Corpus
    from paper_2602_02827_b200.pipeline import stage1_topk

    rng = np.random.default_rng(n_tok + rows)
    x = W._unit(rng.standard_normal((n_tok, d)))
    if dup:
        n = int(dup * n_tok)
        x[rng.integers(0, n_tok, n)] = x[rng.integers(0, n_tok, n)]
    lens = np.full(n_tok // 50, 50)
    lens[-1] += n_tok - lens.sum()
    off = np.concatenate([[0], np.cumsum(lens)])
    corpus = Corpus(_t(W._cast(x, dt), dt), off)
    q = W._unit(rng.standard_normal((rows, d)))
    q[: rows // 4] = x[rng.integers(0, n_tok, rows // 4)]  # exact matches + their duplicates tie
    qt = _t(W._cast(q, dt), dt)
    tok_s, val_s = stage1_topk(corpus, qt, kp, clamp, path="simt")
    tok_t, val_t = stage1_topk(corpus, qt, kp, clamp, path="tc")
    assert stage1_topk.last_paths == ["tc"]
    np.testing.assert_array_equal(tok_t, tok_s)
    np.testing.assert_array_equal(val_t, val_s)
    # values non-increasing, ties ordered by token index
    assert np.all(np.diff(val_s, axis=1) <= 0)
    tie = np.diff(val_s, axis=1) == 0
    assert np.all(np.diff(tok_s, axis=1)[tie] > 0)


def test_tc_scan_hands_zero_ties_to_simt():
    from paper_2602_02827_b200.batch import Corpus
    from paper_2602_02827_b200.pipeline import stage1_topk

    rng = np.random.default_rng(5)
    x = np.abs(W._unit(rng.standard_normal((10_000, 64))))  # all-positive corpus
    off = np.array([0, 4000, 10_000])
    corpus = Corpus(_t(W._cast(x, "f16"), "f16"), off)
    q = -np.abs(W._unit(rng.standard_normal((4, 64))))      # every similarity <= 0 -> clamped zeros
    tok, val = stage1_topk(corpus, _t(W._cast(q, "f16"), "f16"), 5, True, path="tc")
    assert stage1_topk.last_paths == ["tc", "simt"]
    np.testing.assert_array_equal(val, 0.0)
    np.testing.assert_array_equal(tok, np.tile(np.arange(5), (4, 1)))  # zero ties -> corpus order


def _facade(z, meta, fi):
    from paper_2602_02827_b200.reranker import ColBanditReranker

    f = meta["facade"][fi]
    m = meta["cases"][f["corpus_case"]]
    p = f"c{m['case']}_"
    toks, off = z[p + "tokens"], z[p + "offsets"]
    t = _t(toks, m["dtype"])
    corpus = [t[off[i]:off[i + 1]] for i in range(len(off) - 1)]
    est = ColBanditReranker(k=f["k"], k_prime=10, similarity="dot", clamp_negative=f["clamp"],
                            bounds_mode=f["bounds_mode"], random_state=f["random_state"]).fit(corpus)
    qs = [_t(z[f"f{fi}_q{qi}"], m["dtype"]) for qi in range(len(f["outcomes"]))]
    return f, est, qs


@pytest.mark.parametrize("fi", range(5))
def test_reranker_rerank_matches_reference_golden(fi):
    z, meta = _load()
    f, est, qs = _facade(z, meta, fi)
    for qi, want in enumerate(f["outcomes"]):
        o = est.rerank(qs[qi], query_index=qi)
        assert list(o.candidates.doc_indices) == want["cand"]
        assert list(o.doc_indices) == want["doc_indices"]
        assert o.doc_ids == tuple(f"doc{i:04d}" for i in want["doc_indices"])
        assert o.reveals == want["reveals"]
        assert o.coverage == want["coverage"]
        assert [list(x) for x in o.result.reveals] == want["trace"]
        assert o.result.iterations == want["iterations"]
        assert o.result.terminated_by == want["terminated_by"]


@pytest.mark.parametrize("fi", [0, 2, 4])
def test_reranker_predict_batched_matches_reference(fi):
    z, meta = _load()
    f, est, qs = _facade(z, meta, fi)
    assert [list(x) for x in est.predict(qs)] == f["predict"]
    batch = est.rerank_batch(qs)
    for qi, o in enumerate(batch):
        assert [list(x) for x in o.result.reveals] == f["outcomes"][qi]["trace"]


def test_reranker_errors():
    from paper_2602_02827_b200.reranker import ColBanditReranker

    est = ColBanditReranker()
    with pytest.raises(RuntimeError, match="not fitted"):
        est.rerank(np.ones((2, 8), np.float16))
    with pytest.raises(ValueError, match="at least one document"):
        est.fit([])
    with pytest.raises(ValueError, match="disagree on embedding dim"):
        est.fit([np.ones((2, 8), np.float16), np.ones((2, 4), np.float16)])
    with pytest.raises(ValueError, match="bounds_mode"):
        ColBanditReranker(bounds_mode="x").fit([np.ones((2, 8), np.float16)])
    est = ColBanditReranker(similarity="dot").fit([np.ones((2, 8), np.float16)])
    with pytest.raises(ValueError, match="does not match corpus dim"):
        est.rerank(np.ones((2, 4), np.float16))


def test_wide_query_and_large_k_prime_match_the_oracle():
    """The facade with 100-token queries (the paper's multimodal queries reach 100 tokens) and k' = 128 on the
    tcgen05 scan: candidates, ANN bounds and the reveal trace against the oracle restatement of
    ColBanditReranker.rerank (oracle/stage1_ref.rerank, pinned to the reference goldens)."""
    from oracle import stage1_ref
    from paper_2602_02827_b200.pipeline import stage1_topk
    from paper_2602_02827_b200.reranker import ColBanditReranker

    rng = np.random.default_rng(100)
    d, n_docs = 128, 120
    lens = rng.integers(60, 160, n_docs)
    toks = W._unit(rng.standard_normal((int(lens.sum()), d)))
    off = np.concatenate([[0], np.cumsum(lens)])
    stored = W._cast(toks, "f16")
    docs = [stored[off[i]:off[i + 1]] for i in range(n_docs)]
    est = ColBanditReranker(k=8, k_prime=128, similarity="dot", clamp_negative=True, random_state=3).fit(docs)
    docs64 = [W.to_float64(x, "f16") for x in docs]
    for qi in range(2):
        q = W._cast(W._unit(rng.standard_normal((100, d))), "f16")
        o = est.rerank(q, query_index=qi)
        assert stage1_topk.last_paths == ["tc"]
        top, ref, kept = stage1_ref.rerank(W.to_float64(q, "f16"), docs64, k=8, k_prime=128, clamp_negative=True,
                                           random_state=3, query_index=qi)
        assert list(o.candidates.doc_indices) == kept and list(o.doc_indices) == top
        assert [tuple(x) for x in o.result.reveals] == [tuple(x) for x in ref.reveals]
