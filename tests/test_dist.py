"""Multi-process (gloo, world_size 2) tests of the sharding host logic, on CPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_02827_b200.dist import balanced_ranges, merge_topk, sharded_topk


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_balanced_ranges_cover_all_documents_contiguously():
    rng = np.random.default_rng(0)
    lens = rng.integers(16, 512, size=10_000)
    off = np.concatenate([[0], np.cumsum(lens)])
    for world in (1, 2, 3, 4, 8):
        r = balanced_ranges(off, world)
        assert r[0][0] == 0 and r[-1][1] == len(lens)
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        toks = [int(off[b] - off[a]) for a, b in r]
        assert max(toks) - min(toks) <= 2 * 512


def test_merge_topk_orders_by_score_then_id():
    s = np.array([1.0, 3.0, 3.0, 2.0, -np.inf])
    i = np.array([7, 9, 4, 1, -1])
    ms, mi = merge_topk(s, i, 4)
    assert mi.tolist() == [4, 9, 1, 7]
    assert ms.tolist() == [3.0, 3.0, 2.0, 1.0]


def _worker(rank, world, port, scores, k, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = len(scores)
        lo, hi = n * rank // world, n * (rank + 1) // world
        local = torch.tensor(scores[lo:hi])
        ids = torch.arange(lo, hi)
        # local Top-k by (-score, id) — what the device Top-K returns per rank
        order = np.lexsort((ids.numpy(), -local.numpy()))[:k]
        ms, mi = sharded_topk(local[order], ids[order], k)
        out[rank] = (ms.tolist(), mi.tolist())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_doc_sharded_topk_equals_single_process_topk(world):
    rng = np.random.default_rng(3)
    scores = np.round(rng.standard_normal(5000), 2)  # plenty of exact ties across ranks
    k = 100
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, scores, k, out), nprocs=world, join=True)
    ref = np.lexsort((np.arange(len(scores)), -scores))[:k]
    for r in range(world):
        ms, mi = out[r]
        assert mi == ref.tolist()
        np.testing.assert_array_equal(ms, scores[ref])


# ---------------------------------------------------------------- document-sharded Col-Bandit protocol
class _ReplayRun:
    """CPU stand-in for ShardedBanditRun (the device step needs a GPU): replays the oracle trace of a run,
    writing the cells this rank owns into the exchange slots (INT64_MIN elsewhere) and asserting that every
    exchange handed it the owner's value — i.e. it exercises drive() and the all-reduce wiring exactly as
    the device runs use them."""

    def __init__(self, ref, n_rows, own):
        from paper_2602_02827_b200.sharded import NOT_MINE

        self.ref, self.n, self.own = ref, n_rows, own
        self.xchg = torch.full((n_rows,), NOT_MINE, dtype=torch.int64)
        self.pos, self.state, self.exchanges = 0, "start", 0

    def _slot(self, i, v):
        from paper_2602_02827_b200.sharded import NOT_MINE, xchg_key

        return xchg_key(v) if self.own[0] <= i < self.own[1] else NOT_MINE

    def step(self):
        from paper_2602_02827_b200.sharded import xchg_value

        rv = self.ref.reveals
        if self.state == "done":
            return
        if self.state == "warm":
            assert [xchg_value(int(x)) for x in self.xchg[: self.n]] == [v for _, _, v in rv[: self.n]]
            self.pos = self.n
        elif self.state == "reveal":
            assert xchg_value(int(self.xchg[0])) == rv[self.pos][2]
            self.pos += 1
        if self.state == "start":  # epsilon-greedy warm-up: reveals 0..N-1 are one cell per row
            for s in range(self.n):
                self.xchg[s] = self._slot(rv[s][0], rv[s][2])
            self.state = "warm"
            return
        if self.pos == len(rv):
            self.state = "done"
            return
        i, _, v = rv[self.pos]
        self.xchg[0] = self._slot(i, v)
        self.state = "reveal"

    def phase(self):
        from paper_2602_02827_b200 import _lib

        return {"warm": _lib.CBX_SHARD_WARMUP, "reveal": _lib.CBX_SHARD_REVEAL, "done": _lib.CBX_SHARD_DONE}[
            self.state]

    def slots(self, ph):
        from paper_2602_02827_b200 import _lib

        return self.n if ph == _lib.CBX_SHARD_WARMUP else 1

    def result(self):
        return self.ref.reveals[: self.pos]


def _bandit_worker(rank, world, port, cells, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import bandit_ref
        from paper_2602_02827_b200.sharded import allreduce_exchange, drive

        ref = bandit_ref.run(cells, -1.0, 1.0, 5, seed=(0, 7))
        n = cells.shape[0]
        own = (n * rank // world, n * (rank + 1) // world)
        got = drive(_ReplayRun(ref, n, own), allreduce_exchange(), check_every=7)
        out[rank] = (got == ref.reveals, len(got))
    finally:
        dist.destroy_process_group()


def test_doc_sharded_bandit_exchange_protocol_over_gloo():
    rng = np.random.default_rng(11)
    cells = np.clip(rng.standard_normal((120, 16)) * 0.2, -1, 1)
    cells[:10] += 0.3  # a separable top group so the run stops well before exhaustion
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_bandit_worker, args=(2, _free_port(), cells, out), nprocs=2, join=True)
    for r in range(2):
        ok, n = out[r]
        assert ok and n > 120


def test_exchange_keys_order_like_values():
    from paper_2602_02827_b200.sharded import NOT_MINE, xchg_key, xchg_value

    vals = [-np.inf, -3.5, -1e-300, -0.0, 0.0, 5e-324, 0.25, 2.0, np.inf]
    keys = [xchg_key(v) for v in vals]
    assert keys == sorted(keys) and len(set(keys)) == len(keys)
    assert all(k > NOT_MINE for k in keys)
    assert [xchg_value(k) for k in keys] == vals
