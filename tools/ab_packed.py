"""A/B of the packed (resident-corpus) scorer: parity against the contiguous tcgen05 batch and timing.

Run once per libcbx build (CBX_TOOLS=1 CBX_LIB=...); prints one JSON line: packed scores bit-equal to the contiguous
scorer on the same candidates, device ms of the packed rerank call and e2e (host in / host out) ms.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_02827_b200 import workloads as W  # noqa: E402
from paper_2602_02827_b200.batch import Corpus, TokenBatch, maxsim_scores  # noqa: E402

cfg = os.environ.get("CFG", "cfg2")
b, (qo, do, qd) = W.gen_batch_device(cfg)
corpus = Corpus(b.d_tokens, do)
rng = np.random.default_rng(0)
nq = b.n_queries
cand = np.concatenate([qd[q] + rng.permutation(int(qd[q + 1] - qd[q])) for q in range(nq)]).astype(np.int64)
order = os.environ.get("ORDER", "random")  # "sorted": each query's candidates in corpus-row order (locality bound)
if order == "sorted":
    cand = np.concatenate([np.sort(cand[qd[q]:qd[q + 1]]) for q in range(nq)])
cand_t = torch.from_numpy(cand).pin_memory()
qh = b.q_tokens.cpu().pin_memory()
k = 10

# contiguous reference: the same candidates gathered into one batch, scored by the tcgen05 batch path
rows, doff, hoff = corpus.gather(cand)
tb = TokenBatch.from_device(b.q_tokens, b.q_tok_off, rows, doff, b.q_doc_off, host_offsets=(qo, hoff, qd))
ref = maxsim_scores(tb, path="tc").clone()
corpus.rerank_topk(qh, qo, cand_t, qd, k)
torch.cuda.synchronize()
got = corpus._ws["scores"][: len(cand)].clone()
equal = bool(torch.equal(ref, got))
maxdiff = float((ref - got).abs().max())
del rows, doff, tb

for _ in range(3):
    corpus.rerank_topk(qh, qo, cand_t, qd, k)
torch.cuda.synchronize()
n = 20
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record()
for _ in range(n):
    corpus.rerank_topk(qh, qo, cand_t, qd, k, sync=False)
s1.record()
torch.cuda.synchronize()
dev_ms = s0.elapsed_time(s1) / n
t0 = time.perf_counter()
for _ in range(n):
    corpus.rerank_topk(qh, qo, cand_t, qd, k)
e2e_ms = (time.perf_counter() - t0) * 1e3 / n
print(json.dumps({"lib": os.environ.get("CBX_LIB", "default"), "cfg": cfg, "order": order, "scores_bit_equal": equal,
                  "max_abs_diff": maxdiff, "device_ms": dev_ms, "e2e_ms": e2e_ms}))
