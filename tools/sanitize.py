"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize.py [part ...]

parts: p1 (tcgen05 scorer + Top-K, packed corpus scorer), exact (float64 cells), bandit (loop kernel: tree /
scan selection, per-cell bounds, pre-warm, matrix source), shard (host-stepped + mailbox multi-rank launch),
stage1 (tcgen05 scan + refine). Prints one line per part; exits non-zero on a parity failure.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_02827_b200 import workloads as W  # noqa: E402

parts = sys.argv[1:] or ["p1", "exact", "bandit", "shard", "stage1"]
torch.cuda.set_device(0)
case = W.gen_query("cfg2", 0, n_docs=60)
off = case.doc_offsets
docs = [case.doc_tokens[off[i]:off[i + 1]] for i in range(case.n_docs)]

if "p1" in parts:
    from paper_2602_02827_b200.batch import Corpus, TokenBatch, rerank_topk

    b = TokenBatch.from_host([case.query, case.query[:20]], [docs, docs[:30]])
    idx, val, sc = rerank_topk(b, 5)
    c = Corpus(torch.from_numpy(case.doc_tokens).cuda(), off)
    cand = np.arange(case.n_docs)[::-1].copy()
    oi, ov = c.rerank_topk(torch.from_numpy(case.query).pin_memory(), [0, 32], cand, [0, case.n_docs], 5)
    torch.cuda.synchronize()
    print("p1 ok", idx[0].tolist(), oi.tolist())

if "exact" in parts:
    from paper_2602_02827_b200.batch import TokenBatch, exact_cells

    cells, s = exact_cells(TokenBatch.from_host([case.query], [docs]))
    torch.cuda.synchronize()
    print("exact ok", float(s.sum()))

if "bandit" in parts:
    from paper_2602_02827_b200 import BanditConfig, BanditJob, CellBounds, run_batch
    from paper_2602_02827_b200.batch import TokenBatch

    b = TokenBatch.from_host([case.query], [docs])
    rng = np.random.default_rng(0)
    lo = rng.uniform(-1, 0, (60, 32))
    jobs = [BanditJob(BanditConfig(k=5, seed=(0, 0)), 60, 32, 0, 0, (-1.0, 1.0), selection="tree"),
            BanditJob(BanditConfig(k=5, seed=(0, 1), alpha_ef=0.2), 60, 32, 0, 0, (-1.0, 1.0), selection="scan"),
            BanditJob(BanditConfig(k=3, seed=(0, 2), explore_mode="static-warmup", gamma_init=0.1), 60, 32, 0, 0,
                      CellBounds(lo, lo + 1.5))]
    r1 = run_batch(jobs, batch=b, prewarm=True)
    r2 = run_batch(jobs, batch=b, prewarm=False)
    assert all(x.reveals == y.reveals for x, y in zip(r1, r2))
    m = torch.from_numpy(rng.uniform(-1, 1, (40, 100))).cuda()
    r3 = run_batch([BanditJob(BanditConfig(k=4, seed=3), 40, 100, 0, 0, (-1.0, 1.0))], matrix=m)
    print("bandit ok", [len(r.reveals) for r in r1 + r3])

if "shard" in parts:
    from paper_2602_02827_b200 import BanditConfig
    from paper_2602_02827_b200.batch import TokenBatch
    from paper_2602_02827_b200.sharded import ShardedBanditRun, drive, run_local_shards, shard_batch

    cfg = BanditConfig(k=5, seed=(0, 0))
    full = TokenBatch.from_host([case.query], [docs])
    res = run_local_shards(full, [(0, 25), (25, 60)], cfg)
    sb = shard_batch(case.query, case.doc_tokens[off[0]:off[60]], off, (0, 60))
    res1 = drive(ShardedBanditRun(sb, (0, 60), cfg), lambda x, n: None, check_every=8, graph=False)
    assert res[0].reveals == res[1].reveals == res1.reveals
    print("shard ok", len(res1.reveals))

if "stage1" in parts:
    from paper_2602_02827_b200.batch import Corpus
    from paper_2602_02827_b200.pipeline import stage1_topk

    big = W.gen_query("cfg2", 1, n_docs=60)
    c = Corpus(torch.from_numpy(big.doc_tokens).cuda(), big.doc_offsets)
    t1, v1 = stage1_topk(c, torch.from_numpy(big.query).cuda(), 8, True, path="tc")
    t2, v2 = stage1_topk(c, torch.from_numpy(big.query).cuda(), 8, True, path="simt")
    assert np.array_equal(t1, t2) and np.array_equal(v1, v2)
    print("stage1 ok", stage1_topk.last_paths)
