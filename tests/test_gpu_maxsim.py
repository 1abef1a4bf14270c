"""P1 parity on the B200: the dense scorer, the exact cell kernel and the Top-K
against the CPU oracle and the reference's golden vectors.

Tolerances (BASELINE.json north_star): scores within 1e-3 relative for
fp16/bf16 inputs, 1e-5 for fp32; Top-K order bit-exact except where the
reference's scores tie within that tolerance. Exact cells must be bit-equal
to the reference for fp16/bf16 (float64 sums of exact products).
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from helpers import batch_of_cases, case_doc_list, storage_dtype, topk_matches
from oracle import maxsim_ref
from paper_2602_02827_b200 import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _batch_from_arrays(queries, docs, dt, clamp=False):
    from paper_2602_02827_b200.batch import TokenBatch

    return TokenBatch.from_host(queries, docs, dtype=storage_dtype(dt), clamp_negative=clamp)


def _p1_cases():
    z = np.load(os.path.join(GOLDEN, "p1_small.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    for m in meta:
        p = f"c{m['case']}_"
        off = z[p + "offsets"]
        toks = z[p + "tokens"]
        docs = [toks[off[i]:off[i + 1]] for i in range(len(off) - 1)]
        yield m, z[p + "query"], docs, z[p + "cells"], z[p + "scores"], z[p + "topk"].tolist()


def test_exact_cells_bit_equal_to_reference_golden():
    from paper_2602_02827_b200.batch import exact_cells

    for m, q, docs, cells, scores, _ in _p1_cases():
        b = _batch_from_arrays([q], [docs], m["dtype"], m["clamp"])
        got_cells, got_scores = exact_cells(b)
        got_cells = got_cells.cpu().numpy()[:, : q.shape[0]]
        if m["dtype"] == "f32":
            np.testing.assert_allclose(got_cells, cells, rtol=0, atol=2e-15)
            np.testing.assert_allclose(got_scores.cpu().numpy(), scores, rtol=1e-13)
        else:
            np.testing.assert_array_equal(got_cells, cells)
            np.testing.assert_array_equal(got_scores.cpu().numpy(), scores)


@pytest.mark.parametrize("path", ["auto", "simt"])
def test_scores_and_topk_match_reference_golden(path):
    from paper_2602_02827_b200.batch import rerank_topk

    for m, q, docs, cells, scores, topk in _p1_cases():
        b = _batch_from_arrays([q], [docs], m["dtype"], m["clamp"])
        rtol = 1e-5 if (m["dtype"] == "f32" or path == "simt") else 1e-3
        idx, val, got = rerank_topk(b, m["k"], path=path)
        np.testing.assert_allclose(got.double().cpu().numpy(), scores, rtol=rtol, atol=rtol)
        assert topk_matches(idx[0].tolist(), topk, scores, rtol)


CONFIG_FIXTURES = [("cfg1", 0), ("cfg2", 0), ("cfg2", 1), ("cfg2", 2), ("cfg3", 0), ("cfg3", 1), ("cfg5", 0),
                   ("cfg5", 1)]


@pytest.mark.parametrize("name,q", CONFIG_FIXTURES)
def test_config_query_matches_reference_golden(name, q):
    from paper_2602_02827_b200.batch import rerank_topk

    path = os.path.join(GOLDEN, f"{name}_q{q}.npz")
    if not os.path.exists(path):
        pytest.skip("fixture missing")
    z = np.load(path)
    cfg = W.CONFIGS[name]
    case = W.gen_query(name, q)
    b = batch_of_cases([case])
    idx, val, got = rerank_topk(b, cfg.k)
    rtol = 1e-5 if cfg.dtype == "f32" else 1e-3
    np.testing.assert_allclose(got.double().cpu().numpy(), z["scores"], rtol=rtol, atol=0)
    assert topk_matches(idx[0].tolist(), z["topk"].tolist(), z["scores"], rtol)
    # the returned Top-K values are the scores of the returned indices
    np.testing.assert_array_equal(val[0].cpu().numpy(), got.cpu().numpy()[idx[0].cpu().numpy()])


def test_multi_query_batch_with_ragged_lq_matches_oracle():
    """cfg3-style queries (Lq in [16, 48] -> 1 or 2 TMEM lane quadrants) in one batch."""
    from paper_2602_02827_b200.batch import rerank_topk

    cases = [W.gen_query("cfg3", q, n_docs=40) for q in range(6)]
    b = batch_of_cases(cases)
    idx, _, got = rerank_topk(b, 5)
    got = got.double().cpu().numpy()
    off = 0
    for qi, c in enumerate(cases):
        s, t, _ = maxsim_ref.score_query(c.query64(), c.docs64(), 5)
        np.testing.assert_allclose(got[off:off + c.n_docs], s, rtol=1e-3)
        assert topk_matches(idx[qi].tolist(), t, s, 1e-3)
        off += c.n_docs


def _rand_case(rng, n_docs, lq, d, dt, lens):
    q = W._cast(W._unit(rng.standard_normal((lq, d))), dt)
    docs = [W._cast(W._unit(rng.standard_normal((L, d))), dt) for L in lens]
    return q, docs


@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("lq,d", [(1, 64), (32, 128), (33, 128), (64, 256), (100, 96), (128, 128), (7, 512)])
def test_shapes_and_ragged_docs(dt, lq, d):
    """Edge shapes: 1-token docs, docs spanning many tiles and chunks, odd dims, Lq up to 128."""
    from paper_2602_02827_b200.batch import rerank_topk

    rng = np.random.default_rng(lq * 1000 + d)
    lens = [1, 1, 2, 127, 128, 129, 255, 256, 257, 3000] + list(rng.integers(1, 400, size=30))
    q, docs = _rand_case(rng, len(lens), lq, d, dt, lens)
    for clamp in (False, True):
        b = _batch_from_arrays([q], [docs], dt, clamp)
        idx, _, got = rerank_topk(b, 7, path="tc")
        q64 = W.to_float64(q, dt)
        s, t, _ = maxsim_ref.score_query(q64, [W.to_float64(x, dt) for x in docs], 7, clamp)
        np.testing.assert_allclose(got.double().cpu().numpy(), s, rtol=1e-3, atol=1e-3)
        assert topk_matches(idx[0].tolist(), t, s, 1e-3)


def test_queries_without_documents_and_many_queries():
    from paper_2602_02827_b200.batch import maxsim_scores

    rng = np.random.default_rng(5)
    queries, docs = [], []
    for qi in range(40):
        n = 0 if qi % 7 == 3 else int(rng.integers(1, 20))
        q, dl = _rand_case(rng, n, 32, 128, "f16", list(rng.integers(1, 300, size=n)))
        queries.append(q)
        docs.append(dl)
    b = _batch_from_arrays(queries, docs, "f16")
    got = maxsim_scores(b).double().cpu().numpy()
    off = 0
    for q, dl in zip(queries, docs):
        if dl:
            s = maxsim_ref.scores_from_cells(maxsim_ref.cell_matrix(q.astype(np.float64),
                                                                    [x.astype(np.float64) for x in dl]))
            np.testing.assert_allclose(got[off:off + len(dl)], s, rtol=1e-3)
        off += len(dl)


def test_topk_multi_pass_large_pool_and_ties():
    from paper_2602_02827_b200.batch import topk

    rng = np.random.default_rng(11)
    n = 100_000
    scores = np.round(rng.standard_normal(n), 2).astype(np.float32)  # many exact ties
    off = torch.tensor([0, n], dtype=torch.int64, device="cuda")
    s = torch.from_numpy(scores).cuda()
    for k in (1, 100, 1000, 5000):
        idx, val = topk(s, off, k, n)
        ref = np.lexsort((np.arange(n), -scores.astype(np.float64)))[:k]
        assert idx[0].cpu().numpy().tolist() == ref.tolist()
        np.testing.assert_array_equal(val[0].cpu().numpy(), scores[ref])
    s64 = torch.from_numpy(scores.astype(np.float64)).cuda()
    idx, _ = topk(s64, off, 100, n)
    assert idx[0].cpu().numpy().tolist() == np.lexsort((np.arange(n), -scores.astype(np.float64)))[:100].tolist()


def test_invalid_arguments_raise_value_error():
    from paper_2602_02827_b200.batch import rerank_topk

    rng = np.random.default_rng(0)
    q, docs = _rand_case(rng, 3, 8, 64, "f16", [4, 5, 6])
    b = _batch_from_arrays([q], [docs], "f16")
    with pytest.raises(ValueError, match="k exceeds"):
        rerank_topk(b, 4)
    with pytest.raises(ValueError):
        rerank_topk(b, 2, path="bogus")


def test_resident_corpus_rerank_matches_oracle():
    """Corpus (HBM-resident, fit once) + per-call candidate ids: gather kernel + scorer + Top-K."""
    from paper_2602_02827_b200.batch import Corpus

    rng = np.random.default_rng(21)
    d = 128
    lens = rng.integers(1, 400, size=500)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    toks = W._cast(W._unit(rng.standard_normal((int(off[-1]), d))), "f16")
    corpus = Corpus(toks, off)
    queries, cands = [], []
    for q in range(7):
        lq = int(rng.integers(1, 40))
        queries.append(W._cast(W._unit(rng.standard_normal((lq, d))), "f16"))
        n = int(rng.integers(5, 120))
        cands.append(rng.choice(500, size=n, replace=q % 2 == 0))  # duplicates allowed
    qo = np.concatenate([[0], np.cumsum([x.shape[0] for x in queries])]).astype(np.int64)
    co = np.concatenate([[0], np.cumsum([len(c) for c in cands])]).astype(np.int64)
    qt = torch.from_numpy(np.concatenate(queries)).pin_memory()
    k = 5
    docs64 = [W.to_float64(toks[off[i]:off[i + 1]], "f16") for i in range(500)]
    for mode in ("packed", "gather"):
        idx, val = corpus.rerank_topk(qt, qo, np.concatenate(cands), co, k, mode=mode)
        for q in range(7):
            s, t, _ = maxsim_ref.score_query(W.to_float64(queries[q], "f16"), [docs64[c] for c in cands[q]], k)
            assert topk_matches(idx[q].tolist(), t, s, 1e-3), mode
            np.testing.assert_allclose(val[q].numpy(), s[idx[q].numpy()], rtol=1e-3)
        with pytest.raises(IndexError):
            corpus.rerank_topk(qt, qo, np.full(int(co[-1]), 500), co, k, mode=mode)


@pytest.mark.parametrize("dt,d,tail", [("f16", 128, 3), ("bf16", 256, 5), ("f16", 64, 7), ("f16", 512, 1),
                                        ("bf16", 96, 6)])
def test_packed_corpus_every_score_at_the_corpus_end(dt, d, tail):
    """Every packed score (k = pool size) against the oracle when the corpus ends off an 8-row group:
    the interleaved 4-D maps stop at their last whole group, boxes past it take the 8-row 2-D path."""
    from paper_2602_02827_b200.batch import Corpus, to_torch_tokens

    rng = np.random.default_rng(d + tail)
    lens = np.concatenate([rng.integers(1, 300, size=60), [8 * 37 + tail, 40 + tail, tail]])
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    toks = W._cast(W._unit(rng.standard_normal((int(off[-1]), d))), dt)
    corpus = Corpus(toks, off, dtype=storage_dtype(dt))
    n = len(lens)
    nd = 24
    qs = [W._cast(W._unit(rng.standard_normal((int(rng.integers(1, 33)), d))), dt) for _ in range(3)]
    # every pool holds the last three corpus documents, in shuffled positions
    cands = [rng.permutation(np.concatenate([rng.choice(n - 3, nd - 3, replace=False), [n - 3, n - 2, n - 1]]))
             for _ in range(3)]
    qt = torch.cat([to_torch_tokens(q, storage_dtype(dt)) for q in qs]).pin_memory()
    qo = np.concatenate([[0], np.cumsum([q.shape[0] for q in qs])]).astype(np.int64)
    co = np.arange(4, dtype=np.int64) * nd
    idx, val = corpus.rerank_topk(qt, qo, np.concatenate(cands), co, nd)
    docs64 = [W.to_float64(toks[off[i]:off[i + 1]], dt) for i in range(n)]
    for q in range(3):
        s, _, _ = maxsim_ref.score_query(W.to_float64(qs[q], dt), [docs64[c] for c in cands[q]], nd)
        assert sorted(idx[q].tolist()) == list(range(nd))
        np.testing.assert_allclose(val[q].numpy(), s[idx[q].numpy()], rtol=1e-3, atol=1e-3)


@pytest.mark.parametrize("dt,lq,d", [("f16", 32, 128), ("bf16", 48, 128), ("bf16", 64, 256), ("f16", 100, 96)])
def test_packed_corpus_scores_match_oracle_on_config_shapes(dt, lq, d):
    """Packed streaming from the corpus: per-document 8-row alignment, docs across tiles, 1-token docs."""
    from paper_2602_02827_b200.batch import Corpus

    rng = np.random.default_rng(lq + d)
    lens = np.concatenate([[1, 7, 8, 9, 127, 128, 129, 1030, 3000], rng.integers(1, 600, size=300)])
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    toks = W._cast(W._unit(rng.standard_normal((int(off[-1]), d))), dt)
    corpus = Corpus(toks, off, dtype=storage_dtype(dt))
    qs = [W._cast(W._unit(rng.standard_normal((int(rng.integers(1, lq + 1)), d))), dt) for _ in range(5)]
    cands = [rng.permutation(len(lens))[: int(rng.integers(20, 200))] for _ in range(5)]
    from paper_2602_02827_b200.batch import to_torch_tokens

    qt = torch.cat([to_torch_tokens(q, storage_dtype(dt)) for q in qs]).pin_memory()
    qo = np.concatenate([[0], np.cumsum([q.shape[0] for q in qs])]).astype(np.int64)
    co = np.concatenate([[0], np.cumsum([len(c) for c in cands])]).astype(np.int64)
    idx, val = corpus.rerank_topk(qt, qo, np.concatenate(cands), co, 10)
    docs64 = [W.to_float64(toks[off[i]:off[i + 1]], dt) for i in range(len(lens))]
    for q in range(5):
        s, t, _ = maxsim_ref.score_query(W.to_float64(qs[q], dt), [docs64[c] for c in cands[q]], 10)
        assert topk_matches(idx[q].tolist(), t, s, 1e-3)
        np.testing.assert_allclose(val[q].numpy(), s[idx[q].numpy()], rtol=1e-3, atol=1e-3)
