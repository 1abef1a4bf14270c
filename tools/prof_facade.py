"""Where ColBanditReranker.rerank spends its time (host profile + device events) on the cfg4 corpus."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2602_02827_b200 import workloads as W  # noqa: E402
from paper_2602_02827_b200.batch import Corpus  # noqa: E402
from paper_2602_02827_b200.reranker import ColBanditReranker  # noqa: E402

cfg = W.CONFIGS["cfg4"]
b4, (qo, do, qd) = W.gen_batch_device(cfg, n_queries=1, seed=0)
corpus = Corpus(b4.d_tokens, do, clamp_negative=True)
est = ColBanditReranker(k=10, k_prime=10, similarity="dot", clamp_negative=True).fit(corpus)
qh = b4.q_tokens.cpu()
for _ in range(3):
    est.rerank(qh, query_index=0)
torch.cuda.synchronize()
t0 = time.perf_counter()
n = 5
for _ in range(n):
    o = est.rerank(qh, query_index=0)
print(f"rerank: {(time.perf_counter() - t0) * 1e3 / n:.2f} ms per query, {len(o.candidates)} candidates")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    est.rerank(qh, query_index=0)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)

# per-phase cycles of the facade's bandit run (cbx_bandit_set_profile)
import ctypes  # noqa: E402

import numpy as np  # noqa: E402

from paper_2602_02827_b200 import _lib  # noqa: E402

prof = torch.zeros(16, dtype=torch.int64, device="cuda")
_lib.load().cbx_bandit_set_profile(ctypes.c_void_p(prof.data_ptr()))
o = est.rerank(qh, query_index=0)
torch.cuda.synchronize()
_lib.load().cbx_bandit_set_profile(None)
ph = prof.cpu().numpy().astype(np.float64)
names = ["scan", "decide", "reveal", "trees", "warmup", "total", "row_update", "sync", "ru_setup", "ru_welford",
         "ru_exactsum", "ru_interval", "p12", "p13", "p14", "p15"]
it = o.result.iterations
print(f"bandit: {it} iterations, {len(o.result.reveals)} reveals, {ph[5] / 1.965e3:.0f} us at 1.965 GHz; cycles/iteration: "
      + ", ".join(f"{n}={v / it:.0f}" for n, v in zip(names, ph)))
