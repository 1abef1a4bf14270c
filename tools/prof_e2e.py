"""Split of the resident-corpus e2e step: host prep, gather kernel, scorer, Top-K, D2H."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_02827_b200 import workloads as W  # noqa: E402
from paper_2602_02827_b200.batch import Corpus  # noqa: E402

b, (qo, do, qd) = W.gen_batch_device("cfg2")
corpus = Corpus(b.d_tokens, do)
rng = np.random.default_rng(0)
nq = b.n_queries
order = os.environ.get('CAND_ORDER', 'shuffle')
if order == 'shuffle':
    cand = np.concatenate([qd[q] + rng.permutation(int(qd[q + 1] - qd[q])) for q in range(nq)]).astype(np.int64)
else:
    cand = np.arange(int(qd[-1]), dtype=np.int64)
MODE = os.environ.get('MODE', 'packed')
cand_t = torch.from_numpy(cand).pin_memory()
qh = b.q_tokens.cpu().pin_memory()
for _ in range(3):
    corpus.rerank_topk(qh, qo, cand_t, qd, 10, mode=MODE)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as p:
    for _ in range(5):
        corpus.rerank_topk(qh, qo, cand_t, qd, 10, mode=MODE)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=15))
t0 = time.perf_counter()
for _ in range(10):
    corpus.rerank_topk(qh, qo, cand_t, qd, 10, mode=MODE)
print("wall ms/step", (time.perf_counter() - t0) * 100)
