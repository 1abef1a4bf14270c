"""Where the host time of the public bandit call goes (cfg2, 256 runs): prepare / launch / collect, cProfile."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2602_02827_b200 import BanditConfig, BanditJob, run_batch  # noqa: E402
from paper_2602_02827_b200 import workloads as W  # noqa: E402
from paper_2602_02827_b200.bandit import collect, launch_batch, prepare_batch  # noqa: E402

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
b, (qo, do, qd) = W.gen_batch_device(cfg)
jobs = [BanditJob(BanditConfig(k=cfg.k, alpha_ef=a, seed=(0, q)), int(qd[q + 1] - qd[q]), int(qo[q + 1] - qo[q]), q,
                  int(qd[q]), (-1.0, 1.0)) for q in range(b.n_queries) for a in cfg.alphas]
for _ in range(2):
    run_batch(jobs, batch=b)
torch.cuda.synchronize()
for it in range(3):
    t0 = time.perf_counter()
    p = prepare_batch(jobs, batch=b)
    t1 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    raw = launch_batch(p)
    e1.record()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    res = collect(raw, jobs, list(p["results"]))
    t4 = time.perf_counter()
    print(f"prepare {1e3*(t1-t0):.2f} ms, launch {1e3*(t2-t1):.2f}, wait {1e3*(t3-t2):.2f} (device "
          f"{e0.elapsed_time(e1):.2f}), collect {1e3*(t4-t3):.2f}, total {1e3*(t4-t0):.2f}")
t0 = time.perf_counter()
run_batch(jobs, batch=b)
print(f"run_batch {1e3*(time.perf_counter()-t0):.2f} ms")
pr = cProfile.Profile()
pr.enable()
run_batch(jobs, batch=b)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
