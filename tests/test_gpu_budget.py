"""Static-budget baselines and full_rerank on the device against the reference goldens (bit-exact)."""

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


def _oracle(c):
    from paper_2602_02827_b200 import DocTokens, MaxSimOracle, QueryTokens, Similarity
    from paper_2602_02827_b200.batch import to_torch_tokens

    if c["source"] == "matrix":
        return MaxSimOracle.from_matrix(np.array(c["cells"]), value_range=(-0.5, 1.5))
    dt, d = c["dtype"], c["dim"]
    npdt = np.float16 if dt == "f16" else np.uint16
    q = np.frombuffer(bytes.fromhex(c["query_hex"]), dtype=npdt).reshape(-1, d)
    toks = np.frombuffer(bytes.fromhex(c["tokens_hex"]), dtype=npdt).reshape(-1, d)
    off = c["offsets"]
    st = "bf16" if dt == "bf16" else None
    tt = to_torch_tokens(toks, st)
    docs = [DocTokens(f"d{i}", tt[off[i]:off[i + 1]]) for i in range(len(off) - 1)]
    return MaxSimOracle(QueryTokens(to_torch_tokens(q, st)), docs, Similarity("dot", -1.0, 1.0))


def _seed(s):
    return tuple(s) if isinstance(s, list) else s


def test_budget_baselines_match_reference_golden():
    from paper_2602_02827_b200 import CellBounds
    from paper_2602_02827_b200.baselines import doc_top_margin, doc_uniform, full_rerank

    with open(os.path.join(GOLDEN, "budget_small.json")) as f:
        cases = json.load(f)
    for c in cases:
        u = doc_uniform(_oracle(c), c["k"], c["gamma"], seed=_seed(c["seed"]))
        m = doc_top_margin(_oracle(c), CellBounds(np.array(c["lo"]), np.array(c["hi"])), c["k"], c["gamma"])
        for got, want in ((u, c["uniform"]), (m, c["margin"])):
            assert got.topk == want["topk"]
            assert got.coverage == want["coverage"]
            assert [list(x) for x in got.reveals] == want["reveals"]
            assert got.iterations == 0 and got.terminated_by == "budget"
        o = _oracle(c)
        f = full_rerank(o, c["k"])
        cells = np.array(c["cells64"])
        assert f.coverage == 1.0 and len(f.reveals) == cells.size and o.reveal_count == cells.size
        sums = [__import__("math").fsum(r) for r in cells.tolist()]
        assert f.topk == sorted(range(len(sums)), key=lambda i: (-sums[i], i))[: c["k"]]


def test_budget_baseline_errors():
    from paper_2602_02827_b200 import CellBounds, MaxSimOracle
    from paper_2602_02827_b200.baselines import doc_top_margin, doc_uniform

    o = MaxSimOracle.from_matrix(np.zeros((3, 4)))
    with pytest.raises(ValueError, match="gamma must be in"):
        doc_uniform(o, 1, 0.0)
    with pytest.raises(ValueError, match="k must be in"):
        doc_uniform(o, 4, 0.5)
    with pytest.raises(ValueError, match="bounds shape does not match"):
        doc_top_margin(o, CellBounds.uniform(2, 4, -1, 1), 1, 0.5)
