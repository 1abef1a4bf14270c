"""The alpha / budget sweep harness on the device against the reference's frontier rows (exact)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _instances(kind, raw):
    from paper_2602_02827_b200 import CellBounds, DocTokens, MaxSimOracle, QueryTokens, Similarity
    from paper_2602_02827_b200.evaluation import EvalInstance

    out = []
    for qi, r in enumerate(raw):
        if kind == "tokens":
            q = np.frombuffer(bytes.fromhex(r["query_hex"]), dtype=np.float16).reshape(-1, 32)
            t = np.frombuffer(bytes.fromhex(r["tokens_hex"]), dtype=np.float16).reshape(-1, 32)
            off = r["offsets"]
            docs = [DocTokens(f"q{qi}d{i}", t[off[i]:off[i + 1]]) for i in range(len(off) - 1)]
            o = MaxSimOracle(QueryTokens(q), docs, Similarity("dot", -1.0, 1.0))
            b = CellBounds.uniform(o.n_docs, o.n_query_tokens, -1.0, 1.0)
        else:
            o = MaxSimOracle.from_matrix(np.array(r["cells"]), value_range=(-0.2, 1.0))
            b = CellBounds.uniform(o.n_docs, o.n_query_tokens, -0.2, 1.0)
        out.append(EvalInstance(o, b, query_id=f"q{qi}", relevant=frozenset(r["relevant"])))
    return out


@pytest.mark.parametrize("kind", ["tokens", "matrix"])
def test_sweeps_match_reference_frontier(kind, tmp_path):
    from paper_2602_02827_b200 import BanditConfig
    from paper_2602_02827_b200.evaluation import coverage_required, sweep_alpha, sweep_budgets, write_frontier_csv

    with open(os.path.join(GOLDEN, "eval_small.json")) as f:
        g = json.load(f)[kind]
    insts = _instances(kind, g["instances"])
    pts = sweep_alpha(insts, 3, BanditConfig(k=3, seed=(5, 1), epsilon=0.2), grid=(0.001, 0.03, 0.3, 1.0))
    assert [p.row() for p in pts] == g["alpha"]
    assert [p.row() for p in sweep_alpha(insts, 2, None, grid=(0.1, 1.0))] == g["alpha_default"]
    bud = sweep_budgets(insts, 3, grid=(0.1, 0.5, 1.0), seed=4)
    assert [p.row() for p in bud] == g["budgets"]
    best = coverage_required(pts + bud, 0.5)
    assert best is None or best.overlap_at_k >= 0.5
    write_frontier_csv(tmp_path / "f.csv", pts)
    assert (tmp_path / "f.csv").read_text().splitlines()[0].startswith("method,param")
