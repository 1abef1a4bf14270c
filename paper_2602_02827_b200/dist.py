"""Multi-GPU plumbing: query sharding and document sharding with an exact Top-K merge.

One process per GPU (torch.distributed, NCCL on the box, gloo in CPU tests).

* Query sharding (cfg2/3/5): queries are independent; each rank scores its own
  contiguous block of queries. No collective on the data path.
* Document sharding (cfg4: one query, 100k candidates): rank r owns a
  contiguous document range balanced by token count, computes the MaxSim
  scores of its documents and its local Top-K, then ONE all-gather of K
  (score, global id) pairs per rank; every rank merges by (-score, id). The
  merge is exact: a document's score does not depend on which rank computed it
  (the scorer's max is order free and its per-document sum order is fixed), so
  the merged list equals the single-GPU Top-K (BASELINE north_star, SURVEY
  §8(e)).
"""

from __future__ import annotations

import numpy as np

__all__ = ["balanced_ranges", "merge_topk", "sharded_topk"]


def balanced_ranges(doc_offsets, world: int) -> list[tuple[int, int]]:
    """Split documents into `world` contiguous ranges of ~equal token count.

    ``doc_offsets`` is the CSR token offset array [n_docs + 1]; range r holds the
    documents whose first token lies in [r * T / world, (r + 1) * T / world).
    """
    off = np.asarray(doc_offsets, dtype=np.int64)
    n = len(off) - 1
    if world <= 0:
        raise ValueError("world must be positive")
    total = int(off[-1] - off[0])
    cuts = [0]
    for r in range(1, world):
        x = off[0] + (total * r) // world
        cuts.append(int(np.searchsorted(off[:n], x, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.array(cuts))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def merge_topk(scores, ids, k: int):
    """Top-k of gathered (score, id) candidates by (-score, id); pads (-inf, -1) are ignored."""
    import torch

    scores = torch.as_tensor(scores, dtype=torch.float64).flatten()
    ids = torch.as_tensor(ids, dtype=torch.int64).flatten()
    keep = ids >= 0
    scores, ids = scores[keep], ids[keep]
    # two stable sorts: by id, then by -score -> (-score, id) lexicographic order
    o1 = torch.argsort(ids, stable=True)
    scores, ids = scores[o1], ids[o1]
    o2 = torch.argsort(-scores, stable=True)
    return scores[o2][:k], ids[o2][:k]


def sharded_topk(local_scores, local_ids, k: int, group=None):
    """All-gather each rank's local Top-k (score, global id) and merge them on every rank.

    ``local_scores``/``local_ids`` are the rank's local Top-k (fewer than k is
    allowed: the rank pads with (-inf, -1)). Works with NCCL (CUDA tensors) and
    gloo (CPU tensors).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = local_scores.device
    s = torch.full((k,), float("-inf"), dtype=torch.float64, device=dev)
    i = torch.full((k,), -1, dtype=torch.int64, device=dev)
    m = min(k, local_scores.numel())
    s[:m] = local_scores.flatten()[:m].to(torch.float64)
    i[:m] = local_ids.flatten()[:m].to(torch.int64)
    gs = [torch.empty_like(s) for _ in range(world)]
    gi = [torch.empty_like(i) for _ in range(world)]
    dist.all_gather(gs, s, group=group)
    dist.all_gather(gi, i, group=group)
    return merge_topk(torch.cat(gs).cpu(), torch.cat(gi).cpu(), k)
