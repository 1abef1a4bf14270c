"""Profiling driver: the P2 bandit over a device-generated config batch (one CTA per run)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_02827_b200 import BanditConfig, BanditJob, run_batch  # noqa: E402
from paper_2602_02827_b200 import workloads as W  # noqa: E402
from paper_2602_02827_b200.bandit import collect, launch_batch, prepare_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--queries", type=int, default=None)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--phases", action="store_true")
ap.add_argument("--selection", default="auto")
ap.add_argument("--no-prewarm", action="store_true")
ap.add_argument("--prewarm", action="store_true")
ap.add_argument("--row-cache", type=int, default=None, nargs="?", const=2,
                help="the row-cache variant; value = cells a row must have revealed before a reveal fills it")
ap.add_argument("--runs", type=int, default=None, help="runs over the first --queries queries, round robin (footprint test)")
a = ap.parse_args()
cfg = W.CONFIGS[a.config]
b, (qo, do, qd) = W.gen_batch_device(cfg, n_queries=a.queries)
nq = b.n_queries
jobs = []
for r in range(a.runs or nq):
    q = r % nq
    for alpha in cfg.alphas:
        jobs.append(BanditJob(BanditConfig(k=cfg.k, alpha_ef=alpha, seed=(0, q)), int(qd[q + 1] - qd[q]),
                              int(qo[q + 1] - qo[q]), q, int(qd[q]), (-1.0, 1.0), selection=a.selection))
lens = np.diff(do)
prof = None
if a.phases:
    import ctypes
    from paper_2602_02827_b200 import _lib
    prof = torch.zeros(len(jobs) * 16, dtype=torch.int64, device="cuda")
    _lib.load().cbx_bandit_set_profile(ctypes.c_void_p(prof.data_ptr()))
elem = b.d_tokens.element_size()
for it in range(a.iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prep = prepare_batch(jobs, batch=b, prewarm=False if a.no_prewarm else (True if a.prewarm else None),
                         row_cache=False if a.row_cache is None else int(a.row_cache))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    raw = launch_batch(prep)
    e1.record()
    torch.cuda.synchronize()
    host = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    st = {}
    res = collect(raw, jobs, list(prep["results"]), stats=st)
    reveals = sum(len(r.reveals) for r in res)
    iters = sum(r.iterations for r in res)
    gbytes = 0
    for j, r in zip(jobs, res):
        if r.reveals:
            rows = np.array([i for i, _, _ in r.reveals]) + j.row_begin
            gbytes += int(lens[rows].sum()) * b.dim * elem
    cov = np.array([r.coverage for r in res])
    print(f"iter {it}: {len(jobs)} runs, kernel {ms:.2f} ms (host {host*1e3:.1f} ms), reveals {reveals}, "
          f"iterations {iters}, {reveals / ms * 1e3 / 1e6:.2f} M cells/s, gather {gbytes / ms / 1e6:.0f} GB/s, "
          f"coverage mean {cov.mean():.4f} [{cov.min():.4f}, {cov.max():.4f}], "
          f"{iters / ms * 1e3 / 1e6:.3f} M iter/s aggregate"
          + (f", rows filled {int(st['rows_filled'].sum())}" if a.row_cache is not None else ""))
    if prof is not None:
        ph = prof.view(-1, 16).cpu().numpy().astype(np.float64)
        its = np.array([r.iterations for r in res], dtype=np.float64)
        names = ["scan", "decide", "reveal", "trees", "warmup", "total", "row_update", "sync",
                 "ru_setup", "ru_welford", "ru_exactsum", "ru_interval", "p12", "p13", "p14", "p15"]
        per_it = ph[:, :16].sum(0) / its.sum()
        print("  cycles/iteration: " + ", ".join(f"{n}={v:.0f}" for n, v in zip(names, per_it)))
