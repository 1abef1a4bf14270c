"""Profiling driver: the P1 step (scorer + Top-K) on a device-generated config batch."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2602_02827_b200 import workloads as W  # noqa: E402
from paper_2602_02827_b200.batch import maxsim_scores, topk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--queries", type=int, default=None)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
cfg = W.CONFIGS[a.config]
b, _ = W.gen_batch_device(cfg, n_queries=a.queries)
scores = torch.empty(b.n_docs, dtype=torch.float32, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(a.iters):
    ev[0].record()
    maxsim_scores(b, out=scores)
    ev[1].record()
    topk(scores, b.q_doc_off, cfg.k, b.max_q_docs)
    torch.cuda.synchronize()
    gb = b.d_tokens.numel() * b.d_tokens.element_size() / 1e9
    ms = ev[0].elapsed_time(ev[1])
    print(f"iter {i}: scorer {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s")
