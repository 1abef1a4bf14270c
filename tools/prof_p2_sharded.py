"""Profiling driver: the document-sharded bandit (cbx_bandit_shard_step + exchange) against the
single-GPU persistent kernel on one device-generated query (cfg4 by default).

--nccl  : exchange through a 1-rank NCCL process group (the real collective call per iteration)
--sim W : W shards simulated in this process (sequential steps, MAX-combined slots; correctness only)
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_02827_b200 import BanditConfig, BanditJob, _lib, run_batch  # noqa: E402
from paper_2602_02827_b200 import workloads as W  # noqa: E402
from paper_2602_02827_b200.batch import TokenBatch  # noqa: E402
from paper_2602_02827_b200.dist import balanced_ranges  # noqa: E402
from paper_2602_02827_b200.sharded import ShardedBanditRun, allreduce_exchange, drive  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--docs", type=int, default=None)
ap.add_argument("--nccl", action="store_true")
ap.add_argument("--sim", type=int, default=0)
ap.add_argument("--check-every", type=int, default=64)
ap.add_argument("--no-graph", action="store_true")
a = ap.parse_args()
cfg = W.CONFIGS[a.config]
b, (qo, do, qd) = W.gen_batch_device(cfg, n_queries=1, n_docs=a.docs)
N, T = b.n_docs, int(qo[1] - qo[0])
bc = BanditConfig(k=cfg.k, seed=(0, 0))


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    r = fn()
    e1.record()
    torch.cuda.synchronize()
    return r, e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3


single, ms1, _ = timed(lambda: run_batch([BanditJob(bc, N, T, 0, 0, (-1.0, 1.0))], batch=b)[0])
print(f"single-GPU kernel: {N} docs, {single.iterations} iterations, {len(single.reveals)} reveals, "
      f"{ms1:.1f} ms ({ms1 * 1e3 / single.iterations:.2f} us/iteration)", flush=True)

exchange = lambda x, n: None  # noqa: E731
if a.nccl:
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    exchange = allreduce_exchange()
run = ShardedBanditRun(b, (0, N), bc)
res, ms2, wall2 = timed(lambda: drive(run, exchange, a.check_every, graph=not a.no_graph))
print(f"sharded step path (1 rank, {'NCCL all-reduce' if a.nccl else 'no exchange'}, "
      f"{'graphs' if not a.no_graph else 'eager'}): {run.steps} launches, "
      f"{ms2:.1f} ms ({ms2 * 1e3 / res.iterations:.2f} us/iteration), trace equal: {res.reveals == single.reveals}, "
      f"topk equal: {res.topk == single.topk}", flush=True)

if a.sim > 1:
    runs = []
    for lo, hi in balanced_ranges(do, a.sim):
        local = np.zeros(N + 1, np.int64)
        local[lo:hi + 1] = do[lo:hi + 1] - do[lo]
        local[hi + 1:] = do[hi] - do[lo]
        sb = TokenBatch.from_device(b.q_tokens, b.q_tok_off, b.d_tokens[int(do[lo]):int(do[hi])],
                                    torch.from_numpy(local).cuda(), b.q_doc_off, False, host_offsets=(qo, local, qd))
        runs.append(ShardedBanditRun(sb, (lo, hi), bc))
    t0 = time.perf_counter()
    for r in runs:
        r.step()
    while True:
        ph = runs[0].phase()
        if ph == _lib.CBX_SHARD_DONE:
            break
        n = runs[0].slots(ph)
        m = torch.stack([r.xchg[:n] for r in runs]).max(0).values
        for r in runs:
            r.xchg[:n].copy_(m)
            r.step()
    outs = [r.result() for r in runs]
    print(f"{a.sim} simulated shards: traces equal: {all(o.reveals == single.reveals for o in outs)}, "
          f"{time.perf_counter() - t0:.1f} s", flush=True)
if a.nccl:
    dist.destroy_process_group()
