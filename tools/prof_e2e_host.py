"""Host overhead of Corpus.rerank_topk (the bench's e2e call) on cfg2: wall vs device, and a cProfile."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_02827_b200 import workloads as W  # noqa: E402
from paper_2602_02827_b200.batch import Corpus  # noqa: E402

cfg = W.CONFIGS["cfg2"]
batch, (qo, do, qd) = W.gen_batch_device(cfg)
corpus = Corpus(batch.d_tokens, do)
nq = batch.n_queries
rng = np.random.default_rng(1234)
cand = np.concatenate([qd[q] + rng.permutation(int(qd[q + 1] - qd[q])) for q in range(nq)]).astype(np.int64)
cand_t = torch.from_numpy(cand).pin_memory()
q_host = batch.q_tokens.cpu().pin_memory()
for _ in range(3):
    corpus.rerank_topk(q_host, qo, cand_t, qd, 10)
torch.cuda.synchronize()
n = 20
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record(s)
for _ in range(n):
    corpus.rerank_topk(q_host, qo, cand_t, qd, 10)
e1.record(s)
torch.cuda.synchronize()
print(f"wall {(time.perf_counter() - t0) * 1e3 / n:.3f} ms/call, events {e0.elapsed_time(e1) / n:.3f} ms/call")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    corpus.rerank_topk(q_host, qo, cand_t, qd, 10)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
