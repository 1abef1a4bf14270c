"""cfg4 — one query against 100,000 candidates (Lq 32, d 128, fp16, K 100) — against the reference.

The golden (tests/golden/cfg4_q0.npz, tests/golden/make_golden.py cfg4) is the unmodified reference's
output on workloads.gen_query("cfg4", 0): exactly rounded P1 scores, the exact Top-100, and the full
Col-Bandit trace of bandit.run (222,088 iterations, 322,086 reveals). Checked here:

* P1: tcgen05 fp32 scores within 1e-3 relative; the float64 cell kernel's fsum scores bit-equal; the exact
  Top-100 identical, the fp32 Top-100 identical except within-tolerance ties; the document-sharded Top-100
  (2/4/8 shards, local Top-100 + merge by (-score, id)) equal to the 1-GPU list with
  bit-equal per-document scores;
* P2: the single-GPU persistent kernel reproduces the trace reveal for reveal (bit-equal values) with the
  same Top-100, iterations, stop reason and coverage; so do the document-sharded runs.
"""

import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN
from helpers import topk_matches
from paper_2602_02827_b200 import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

PATH = os.path.join(GOLDEN, "cfg4_q0.npz")


def _fingerprint(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def cfg4():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(PATH):
        pytest.skip("cfg4 golden missing")
    torch.cuda.set_device(0)
    from paper_2602_02827_b200.batch import TokenBatch

    z = dict(np.load(PATH))
    case = W.gen_query("cfg4", 0)
    assert _fingerprint(case.query, case.doc_tokens, case.doc_offsets) == bytes(z["fingerprint"]).decode()
    off = case.doc_offsets
    q = torch.from_numpy(case.query).cuda()
    toks = torch.from_numpy(case.doc_tokens).cuda()
    b = TokenBatch.from_device(q, torch.tensor([0, q.shape[0]], device="cuda"), toks, torch.from_numpy(off).cuda(),
                               torch.tensor([0, case.n_docs], device="cuda"), False,
                               host_offsets=(np.array([0, q.shape[0]]), off, np.array([0, case.n_docs])))
    return case, b, z


def test_p1_scores_and_top100(cfg4):
    from paper_2602_02827_b200.batch import exact_cells, maxsim_scores, topk

    case, b, z = cfg4
    ref = z["scores"]
    s32 = maxsim_scores(b)
    np.testing.assert_allclose(s32.double().cpu().numpy(), ref, rtol=1e-3, atol=0)
    cells, s64 = exact_cells(b)
    np.testing.assert_array_equal(s64.cpu().numpy(), ref)  # bit-equal math.fsum of the float64 cells
    K = W.CONFIGS["cfg4"].k
    exact = topk(s64, b.q_doc_off, K, b.n_docs)[0].cpu().numpy().ravel().tolist()
    assert exact == z["topk"].tolist()
    fast = topk(s32, b.q_doc_off, K, b.n_docs)[0].cpu().numpy().ravel().tolist()
    assert topk_matches(fast, z["topk"].tolist(), ref, 1e-3)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_p1_document_sharded_top100(cfg4, world):
    from paper_2602_02827_b200.batch import TokenBatch, maxsim_scores, topk
    from paper_2602_02827_b200.dist import balanced_ranges, merge_topk

    case, b, z = cfg4
    K = W.CONFIGS["cfg4"].k
    full = maxsim_scores(b).cpu()
    off = case.doc_offsets
    gs, gi = [], []
    for lo, hi in balanced_ranges(off, world):
        local = (off[lo:hi + 1] - off[lo]).astype(np.int64)
        sb = TokenBatch.from_device(b.q_tokens, b.q_tok_off, b.d_tokens[int(off[lo]):int(off[hi])],
                                    torch.from_numpy(local).cuda(), torch.tensor([0, hi - lo], device="cuda"), False,
                                    host_offsets=(np.array([0, 32]), local, np.array([0, hi - lo])))
        s = maxsim_scores(sb)
        assert torch.equal(s.cpu(), full[lo:hi])  # a document's score does not depend on its shard
        i, v = topk(s, sb.q_doc_off, K, hi - lo)
        gs.append(v.cpu().view(-1).double())
        gi.append(i.cpu().view(-1).to(torch.int64) + lo)
    _, ids = merge_topk(torch.cat(gs), torch.cat(gi), K)
    single = topk(full.cuda(), b.q_doc_off, K, b.n_docs)[0].cpu().view(-1).tolist()
    assert ids.tolist() == single
    assert topk_matches(single, z["topk"].tolist(), z["scores"], 1e-3)


def _assert_trace(res, z):
    got = np.array([(i, t) for i, t in zip(res.reveals.i, res.reveals.t)], dtype=np.int32).reshape(-1, 2) \
        if hasattr(res.reveals, "i") else np.array([(i, t) for i, t, _ in res.reveals], np.int32).reshape(-1, 2)
    exp = z["a0_trace_it"]
    assert got.shape == exp.shape
    np.testing.assert_array_equal(got, exp)
    vals = res.reveals.v if hasattr(res.reveals, "v") else np.array([v for *_, v in res.reveals])
    np.testing.assert_array_equal(vals, z["a0_trace_v"])
    assert res.topk == z["a0_topk"].tolist()
    cov, iters, sep = z["a0_stats"]
    assert res.coverage == cov and res.iterations == int(iters)
    assert res.terminated_by == ("separation" if sep else "exhaustion")


@pytest.mark.parametrize("row_cache", [False, True])
def test_p2_single_gpu_trace(cfg4, row_cache):
    from paper_2602_02827_b200 import BanditConfig, BanditJob, run_batch

    case, b, z = cfg4
    cfg = W.CONFIGS["cfg4"]
    res = run_batch([BanditJob(BanditConfig(k=cfg.k, seed=(0, 0)), case.n_docs, 32, 0, 0, (-1.0, 1.0))], batch=b,
                    row_cache=row_cache)[0]
    _assert_trace(res, z)


def test_p2_sharded_one_rank_trace(cfg4):
    """The host-stepped shard protocol (cbx_bandit_shard_step + exchange per iteration) at one rank."""
    from paper_2602_02827_b200 import BanditConfig
    from paper_2602_02827_b200.sharded import ShardedBanditRun, drive

    case, b, z = cfg4
    run = ShardedBanditRun(b, (0, case.n_docs), BanditConfig(k=W.CONFIGS["cfg4"].k, seed=(0, 0)))
    _assert_trace(drive(run, lambda x, n: None), z)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_p2_mailbox_sharded_trace(cfg4, world):
    """The persistent document-sharded run (one launch, `world` rank CTAs exchanging every revealed cell
    through device-memory inboxes) reproduces the reference trace on every rank."""
    from paper_2602_02827_b200 import BanditConfig
    from paper_2602_02827_b200.dist import balanced_ranges
    from paper_2602_02827_b200.sharded import run_local_shards

    case, b, z = cfg4
    res = run_local_shards(b, balanced_ranges(case.doc_offsets, world),
                           BanditConfig(k=W.CONFIGS["cfg4"].k, seed=(0, 0)))
    for r in res:
        _assert_trace(r, z)
