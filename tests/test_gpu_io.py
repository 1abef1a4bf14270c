"""Loading CBM1 manifests / CBH1 matrices straight into device memory, then reranking from them."""

import numpy as np
import pytest

from paper_2602_02827_b200 import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def test_load_corpus_then_rerank_matches_oracle(tmp_path):
    from oracle import stage1_ref
    from paper_2602_02827_b200 import io as cio
    from paper_2602_02827_b200.reranker import ColBanditReranker

    rng = np.random.default_rng(11)
    docs = [W._unit(rng.standard_normal((int(rng.integers(1, 40)), 32))).astype(np.float16).astype(np.float64)
            for _ in range(60)]
    entries = []
    for i, d in enumerate(docs):
        cio.write_vectors(tmp_path / f"d{i}.cbm", d)
        entries.append((f"doc-{i}", f"d{i}.cbm"))
    cio.write_manifest(tmp_path / "corpus.jsonl", entries)
    corpus = cio.load_corpus(tmp_path / "corpus.jsonl")
    assert corpus.doc_ids == [e[0] for e in entries] and corpus.tokens.dtype == torch.float32
    np.testing.assert_array_equal(corpus.tokens.double().cpu().numpy(), np.concatenate(docs))
    q = W._unit(rng.standard_normal((9, 32))).astype(np.float16).astype(np.float64)
    est = ColBanditReranker(k=4, k_prime=6, similarity="dot", clamp_negative=True).fit(corpus)
    out = est.rerank(q.astype(np.float32), query_index=2)
    top, res, kept = stage1_ref.rerank(q, docs, k=4, k_prime=6, clamp_negative=True, query_index=2)
    assert list(out.candidates.doc_indices) == kept
    assert list(out.doc_indices) == top and out.doc_ids == tuple(f"doc-{i}" for i in top)
    assert [tuple(x) for x in out.result.reveals] == [tuple(x) for x in res.reveals]


def test_load_matrix_oracle(tmp_path):
    from paper_2602_02827_b200 import BanditConfig, CellBounds, run
    from paper_2602_02827_b200 import io as cio
    from oracle import bandit_ref

    m = np.random.default_rng(2).uniform(-0.2, 1.0, size=(30, 12))
    cio.write_matrix(tmp_path / "h.cbh", m)
    o = cio.load_matrix_oracle(tmp_path / "h.cbh", value_range=(-0.5, 1.5))
    m32 = m.astype(np.float32).astype(np.float64)
    np.testing.assert_array_equal(o.row_values(3), m32[3])
    got = run(o, CellBounds.uniform(30, 12, -0.5, 1.5), BanditConfig(k=4, seed=9))
    ref = bandit_ref.run(m32, -0.5, 1.5, 4, seed=9)
    assert got.topk == ref.topk and [tuple(x) for x in got.reveals] == [tuple(x) for x in ref.reveals]
