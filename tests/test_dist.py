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
