"""Document-sharded Col-Bandit on the B200 (SURVEY §8(e), cfg4's multi-GPU path).

The test box has one GPU, so the ranks are simulated in one process: each
shard is its own ShardedBanditRun holding only its documents' tokens, the
shards step one after another (no kernel waits on another) and the exchange is
the element-wise MAX that the NCCL all-reduce computes across ranks. Every
shard must reproduce the single-GPU trace reveal for reveal, and the single-GPU
trace must match the oracle restatement of bandit.run.
"""

import numpy as np
import pytest

from helpers import case_doc_list
from oracle import bandit_ref, maxsim_ref
from paper_2602_02827_b200 import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def drive_shards(runs):
    """In-process stand-in for drive() over len(runs) ranks: step all, MAX-combine the slots, repeat."""
    from paper_2602_02827_b200 import _lib

    for r in runs:
        r.step()
    while True:
        phases = {r.phase() for r in runs}
        assert len(phases) == 1, phases  # replicated state: every rank is at the same exchange
        ph = phases.pop()
        if ph == _lib.CBX_SHARD_DONE:
            return [r.result() for r in runs]
        n = runs[0].slots(ph)
        m = torch.stack([r.xchg[:n] for r in runs]).max(0).values
        for r in runs:
            r.xchg[:n].copy_(m)
            r.step()


def _pool(n_docs, q=0, cfg="cfg4"):
    case = W.gen_query(cfg, q, n_docs=n_docs)
    return case, case_doc_list(case)


def _shard_runs(case, docs, world, cfg, bounds=(-1.0, 1.0)):
    from paper_2602_02827_b200.dist import balanced_ranges
    from paper_2602_02827_b200.sharded import ShardedBanditRun, shard_batch

    off = case.doc_offsets
    runs = []
    for lo, hi in balanced_ranges(off, world):
        toks = case.doc_tokens[off[lo]:off[hi]]
        b = shard_batch(case.query, toks, off, (lo, hi))
        runs.append(ShardedBanditRun(b, (lo, hi), cfg, bounds))
    return runs


def _single(case, docs, cfg, bounds=(-1.0, 1.0)):
    from paper_2602_02827_b200 import BanditJob, run_batch
    from paper_2602_02827_b200.batch import TokenBatch

    b = TokenBatch.from_host([case.query], [docs])
    return run_batch([BanditJob(cfg, case.n_docs, case.query.shape[0], 0, 0, bounds)], batch=b)[0]


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_trace_equals_single_gpu_and_oracle(world):
    from paper_2602_02827_b200 import BanditConfig

    case, docs = _pool(600)
    cfg = BanditConfig(k=10, seed=(0, 0))
    single = _single(case, docs, cfg)
    cells = maxsim_ref.cell_matrix(case.query64(), case.docs64())
    ref = bandit_ref.run(cells, -1.0, 1.0, 10, seed=(0, 0))
    assert [tuple(x) for x in single.reveals] == [tuple(x) for x in ref.reveals]
    for res in drive_shards(_shard_runs(case, docs, world, cfg)):
        assert res.reveals == single.reveals
        assert res.topk == single.topk
        assert (res.iterations, res.terminated_by, res.coverage) == (
            single.iterations, single.terminated_by, single.coverage)


@pytest.mark.parametrize("mode", ["static-warmup", "uniform-row"])
def test_sharded_other_explore_modes(mode):
    from paper_2602_02827_b200 import BanditConfig

    case, docs = _pool(300, q=1)
    cfg = BanditConfig(k=5, seed=(0, 1), explore_mode=mode, gamma_init=0.05, alpha_ef=0.3)
    single = _single(case, docs, cfg)
    for res in drive_shards(_shard_runs(case, docs, 2, cfg)):
        assert res.reveals == single.reveals and res.topk == single.topk


def test_sharded_per_cell_bounds():
    from paper_2602_02827_b200 import BanditConfig, CellBounds

    case, docs = _pool(300, q=2)
    cells = maxsim_ref.cell_matrix(case.query64(), case.docs64())
    rng = np.random.default_rng(5)
    lo = cells - rng.uniform(0.0, 0.3, cells.shape)
    hi = cells + rng.uniform(0.0, 0.3, cells.shape)
    bounds = CellBounds(lo, hi)
    cfg = BanditConfig(k=5, seed=(0, 2))
    single = _single(case, docs, cfg, bounds)
    ref = bandit_ref.run(cells, lo, hi, 5, seed=(0, 2))
    assert [tuple(x) for x in single.reveals] == [tuple(x) for x in ref.reveals]
    for res in drive_shards(_shard_runs(case, docs, 2, cfg, bounds)):
        assert res.reveals == single.reveals and res.topk == single.topk


def test_drive_with_a_one_rank_group_matches_single_gpu():
    """The production driver (batched reveal exchanges between host syncs) with a no-op exchange."""
    from paper_2602_02827_b200 import BanditConfig
    from paper_2602_02827_b200.sharded import drive

    case, docs = _pool(400, q=3)
    cfg = BanditConfig(k=10, seed=(0, 3))
    single = _single(case, docs, cfg)
    (run,) = _shard_runs(case, docs, 1, cfg)
    res = drive(run, lambda xchg, n: None, check_every=16)
    assert res.reveals == single.reveals and res.topk == single.topk


# ---------------------------------------------------------------- the persistent mailbox exchange
def _full_batch(case, docs):
    from paper_2602_02827_b200.batch import TokenBatch

    return TokenBatch.from_host([case.query], [docs])


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_mailbox_ranks_in_one_launch_match_single_gpu(world):
    """cbx_bandit_shard_run with `world` co-resident rank CTAs exchanging through device-memory inboxes:
    every rank's trace equals the single-GPU kernel's and the oracle's."""
    from paper_2602_02827_b200 import BanditConfig
    from paper_2602_02827_b200.dist import balanced_ranges
    from paper_2602_02827_b200.sharded import run_local_shards

    case, docs = _pool(600)
    cfg = BanditConfig(k=10, seed=(0, 0))
    single = _single(case, docs, cfg)
    cells = maxsim_ref.cell_matrix(case.query64(), case.docs64())
    ref = bandit_ref.run(cells, -1.0, 1.0, 10, seed=(0, 0))
    assert single.reveals == ref.reveals
    res = run_local_shards(_full_batch(case, docs), balanced_ranges(case.doc_offsets, world), cfg)
    assert len(res) == world
    for r in res:
        assert r.reveals == single.reveals and r.topk == single.topk
        assert (r.iterations, r.terminated_by, r.coverage) == (single.iterations, single.terminated_by,
                                                               single.coverage)


@pytest.mark.parametrize("mode", ["static-warmup", "uniform-row"])
def test_mailbox_other_explore_modes_and_per_cell_bounds(mode):
    from paper_2602_02827_b200 import BanditConfig, CellBounds
    from paper_2602_02827_b200.dist import balanced_ranges
    from paper_2602_02827_b200.sharded import run_local_shards

    case, docs = _pool(300, q=1)
    cells = maxsim_ref.cell_matrix(case.query64(), case.docs64())
    rng = np.random.default_rng(7)
    bounds = CellBounds(cells - rng.uniform(0.0, 0.3, cells.shape), cells + rng.uniform(0.0, 0.3, cells.shape))
    cfg = BanditConfig(k=5, seed=(0, 1), explore_mode=mode, gamma_init=0.05, alpha_ef=0.3)
    for bnd in ((-1.0, 1.0), bounds):
        single = _single(case, docs, cfg, bnd)
        for r in run_local_shards(_full_batch(case, docs), balanced_ranges(case.doc_offsets, 3), cfg, bnd):
            assert r.reveals == single.reveals and r.topk == single.topk
