"""Drop-in Stage-1 retrieval (colbandit/pipeline.py) on the B200.

``generate_candidates`` keeps the reference's arguments, result types,
ordering and error messages (pipeline.py:105-158): per query token the
``k_prime`` corpus tokens of highest similarity, ties to the earlier corpus
token; candidates are the owners of kept tokens in corpus order;
``exact_cells`` holds each surfaced (candidate, token) pair's exact row
maximum. The scan is ``cbx_stage1_topk`` (csrc/stage1.cu: one tcgen05 pass
over the HBM-resident corpus + float64 refine for fp16/bf16 corpora, float64
CUDA-core scan otherwise) and the exact row maxima come from the float64
cell kernel over the gathered candidate pool — the same fma order as the
scan, so a bound recorded as exact equals the later reveal bit for bit.
``derive_bounds`` and the JSON artifact helpers are host-side bookkeeping
(pipeline.py:161-230).
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

import numpy as np

from . import _lib
from .bounds import CellBounds
from .oracle import DocTokens, QueryTokens, Similarity

__all__ = ["TokenNeighbor", "TokenNeighborList", "CandidateSet", "generate_candidates", "derive_bounds",
           "save_candidates", "load_candidates", "stage1_topk", "Stage1Result", "stage1"]

CANDIDATES_FORMAT = "colbandit-candidates-v1"
_S1_PATHS = {"auto": _lib.CBX_PATH_AUTO, "tc": _lib.CBX_PATH_TC, "tcgen05": _lib.CBX_PATH_TC,
             "simt": _lib.CBX_PATH_SIMT}


@dataclass(frozen=True)
class TokenNeighbor:
    """pipeline.py:43-50."""

    doc_id: str
    doc_index: int
    token_index: int
    similarity: float


@dataclass(frozen=True)
class TokenNeighborList:
    """pipeline.py:53-68."""

    token: int
    neighbors: tuple[TokenNeighbor, ...]

    def __post_init__(self) -> None:
        sims = [nb.similarity for nb in self.neighbors]
        if any(a < b for a, b in zip(sims, sims[1:])):
            raise ValueError(f"token {self.token}: neighbor similarities must be non-increasing")

    @property
    def kth_similarity(self) -> float:
        return self.neighbors[-1].similarity


@dataclass(frozen=True)
class CandidateSet:
    """pipeline.py:71-90."""

    doc_ids: tuple[str, ...]
    doc_indices: tuple[int, ...]
    exact_cells: dict[tuple[int, int], float]

    def __post_init__(self) -> None:
        if len(self.doc_ids) != len(self.doc_indices):
            raise ValueError("doc_ids and doc_indices must align")
        if len(set(self.doc_ids)) != len(self.doc_ids):
            raise ValueError("candidate doc_ids must be distinct")

    def __len__(self) -> int:
        return len(self.doc_ids)


# ---------------------------------------------------------------- device scan
def _rows_in(corpus, rows):
    """Query rows as a device tensor in the corpus dtype when that is lossless, else (rows, widened corpus)."""
    import torch

    from .batch import to_torch_tokens

    t = rows if isinstance(rows, torch.Tensor) else to_torch_tokens(rows)
    cd = corpus.tokens.dtype
    if t.dtype == cd:
        return t.to(corpus.tokens.device), corpus
    cast = t.to(cd)
    if torch.equal(cast.to(torch.float64).cpu(), t.to(torch.float64).cpu()):
        return cast.to(corpus.tokens.device), corpus
    wide = torch.float64 if torch.float64 in (t.dtype, cd) else torch.float32
    return t.to(wide).to(corpus.tokens.device), corpus.widened(wide)


def stage1_topk(corpus, rows, k_prime: int, clamp_negative: bool, path: str = "auto"):
    """Device Stage-1 scan: (token index [R, k], similarity [R, k]) numpy arrays, k = min(k_prime, corpus tokens).

    ``rows`` [R, dim] are the query-token rows (any number of queries, R <= 65535). A tcgen05 scan that
    reports a list overflow or zero ties is re-run on the float64 CUDA-core path (still on the device).
    """
    torch = _lib.require_cuda()
    lib = _lib.load()
    from .batch import dtype_code

    if path not in _S1_PATHS:
        raise ValueError(f"path must be one of {sorted(_S1_PATHS)}, got {path!r}")
    q, corp = _rows_in(corpus, rows)
    q = q.contiguous()
    R = int(q.shape[0])
    kk = min(int(k_prime), corp.n_tokens)
    s = _lib.CbxBatch()
    s.q_tokens, s.n_q_tokens = q.data_ptr(), R
    s.d_tokens, s.n_d_tokens = corp.tokens.data_ptr(), corp.n_tokens
    s.dim, s.dtype, s.clamp_negative = corp.dim, dtype_code(corp.tokens.dtype), int(bool(clamp_negative))
    s.max_lq = R
    dev = corp.tokens.device
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    eff = _S1_PATHS[path]
    if eff == _lib.CBX_PATH_AUTO:
        eff = _lib.CBX_PATH_TC if _tc_eligible(corp, kk) else _lib.CBX_PATH_SIMT
    tried = []
    while True:
        wsb = lib.cbx_stage1_workspace_bytes(ctypes.byref(s), kk, eff)
        norm = corp.norm_max() if eff == _lib.CBX_PATH_TC else 0.0
        ws = torch.empty(max(int(wsb), 1), dtype=torch.uint8, device=dev)
        tok = torch.empty((R, kk), dtype=torch.int64, device=dev)
        val = torch.empty((R, kk), dtype=torch.float64, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.check(lib.cbx_stage1_topk(ctypes.byref(s), kk, eff, ctypes.c_float(norm), tok.data_ptr(),
                                       val.data_ptr(), status.data_ptr(), ws.data_ptr(), int(wsb), stream),
                   "stage1")
        st = int(status.item())
        tried.append("tc" if eff == _lib.CBX_PATH_TC else "simt")
        if st == 0 or eff == _lib.CBX_PATH_SIMT:
            break
        eff = _lib.CBX_PATH_SIMT  # list overflow / zero ties: the float64 CUDA-core scan decides
    stage1_topk.last_paths = tried
    return tok.cpu().numpy(), val.cpu().numpy()


def _tc_fits(dim: int, kk: int) -> bool:
    """The tcgen05 scan's shared memory for k' (mirrors tc_fits in csrc/stage1.cu): query block, k' sorted
    tops per row, scratch and at least two tile stages within 227 KB."""
    kb = (dim + 63) // 64
    fixed = 1024 + kb * 16384 + 4 * kk * 128 + 4 * 32 * 128 + 8 * 32
    if fixed >= 227 * 1024:
        return False
    budget = 227 * 1024 - fixed
    tile_n = 128 if budget // (kb * 16384) >= 3 else 64
    return budget // (kb * tile_n * 128) >= 2


def _tc_eligible(corpus, kk) -> bool:
    import torch

    return (corpus.tokens.dtype in (torch.float16, torch.bfloat16) and corpus.dim % 8 == 0 and corpus.dim <= 256
            and kk <= 256 and _tc_fits(corpus.dim, kk) and corpus.n_tokens >= 8192)


@dataclass
class Stage1Result:
    """Stage-1 output of one query."""

    candidates: CandidateSet
    neighbor_lists: list


def _neighbors_of(corpus, tok_row: np.ndarray, val_row: np.ndarray, t: int, doc_ids) -> TokenNeighborList:
    doc = np.searchsorted(corpus.offsets_host, tok_row, side="right") - 1
    nbs = tuple(TokenNeighbor(doc_ids[int(d)], int(d), int(g - corpus.offsets_host[d]), float(v))
                for g, d, v in zip(tok_row, doc, val_row))
    return TokenNeighborList(t, nbs)


def stage1(corpus, queries: Sequence, k_prime: int, clamp_negative: bool, path: str = "auto"):
    """Stage 1 for many queries in one device scan.

    Returns ``(results, pool_batch)``: per query a :class:`Stage1Result`, and one device TokenBatch whose
    query ``i`` owns the candidate pool of query ``i`` (gathered from the corpus on device, corpus order) —
    the cell source of the adaptive stage. The surfaced pairs' exact row maxima come from one float64 cell
    launch over that batch.
    """
    import torch

    from .batch import TokenBatch, exact_cells, to_torch_tokens

    if k_prime < 1:
        raise ValueError(f"k_prime must be at least 1, got {k_prime}")
    rows = [q._store if isinstance(q, QueryTokens) else to_torch_tokens(q) for q in queries]
    if not rows:
        return [], None
    lq = [int(r.shape[0]) for r in rows]
    if len({r.dtype for r in rows}) > 1:
        rows = [r.to(torch.float64) for r in rows]
    allrows, corp = _rows_in(corpus, torch.cat([r.cpu() for r in rows]))
    allrows = allrows.contiguous()
    toks, vals = [], []
    for a in range(0, allrows.shape[0], 65535):
        tk, vl = stage1_topk(corp, allrows[a:a + 65535], k_prime, clamp_negative, path)
        toks.append(tk)
        vals.append(vl)
    tok = np.concatenate(toks)
    val = np.concatenate(vals)
    doc_ids = corpus.doc_ids or [f"doc{i:04d}" for i in range(corpus.n_docs)]
    meta = []
    r0 = 0
    for n in lq:
        nls = [_neighbors_of(corpus, tok[r0 + t], val[r0 + t], t, doc_ids) for t in range(n)]
        r0 += n
        hit_docs = sorted({nb.doc_index for nl in nls for nb in nl.neighbors})
        hit_pairs = sorted({(nb.doc_index, nl.token) for nl in nls for nb in nl.neighbors})
        meta.append((nls, hit_docs, hit_pairs))
    pool_ids = np.concatenate([np.asarray(m[1], np.int64) for m in meta])
    rows_dev, off_dev, off_host = corp.gather(pool_ids)
    qd = np.zeros(len(rows) + 1, np.int64)
    np.cumsum([len(m[1]) for m in meta], out=qd[1:])
    qo = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(lq, out=qo[1:])
    dev = rows_dev.device
    b = TokenBatch.from_device(allrows, torch.from_numpy(qo).to(dev), rows_dev, off_dev,
                               torch.from_numpy(qd).to(dev), clamp_negative, host_offsets=(qo, off_host, qd))
    cells, _ = exact_cells(b, with_scores=False)
    cells = cells.cpu().numpy()
    results = []
    for qi, (nls, hit_docs, hit_pairs) in enumerate(meta):
        row_of = {di: r for r, di in enumerate(hit_docs)}
        base = int(qd[qi])
        exact = {(row_of[di], t): float(cells[base + row_of[di], t]) for di, t in hit_pairs}
        cand = CandidateSet(tuple(doc_ids[d] for d in hit_docs), tuple(int(d) for d in hit_docs), exact)
        results.append(Stage1Result(cand, nls))
    return results, b


# ---------------------------------------------------------------- reference API
def generate_candidates(query: QueryTokens, corpus, similarity: Similarity, k_prime: int,
                        path: str = "auto") -> tuple[CandidateSet, list[TokenNeighborList]]:
    """pipeline.py:105-158 — the Stage-1 scan (device). ``corpus``: list of DocTokens or a batch.Corpus."""
    from .batch import Corpus

    if corpus is None or (not isinstance(corpus, Corpus) and len(corpus) == 0):
        raise ValueError("corpus must contain at least one document")
    if k_prime < 1:
        raise ValueError(f"k_prime must be at least 1, got {k_prime}")
    dev_corpus = corpus if isinstance(corpus, Corpus) else Corpus.from_docs(list(corpus))
    r = stage1(dev_corpus, [query], k_prime, similarity.clamp_negative, path)[0][0]
    return r.candidates, r.neighbor_lists


def derive_bounds(candidates: CandidateSet, neighbor_lists: list[TokenNeighborList],
                  similarity: Similarity) -> CellBounds:
    """pipeline.py:161-185 — floor = similarity floor; ceiling = exact row max where surfaced, else k'-th sim."""
    n = len(candidates)
    n_tokens = len(neighbor_lists)
    if n == 0 or n_tokens == 0:
        raise ValueError("need at least one candidate and one query token")
    lo = np.full((n, n_tokens), similarity.range_lo, dtype=np.float64)
    hi = np.repeat(np.array([[nl.kth_similarity for nl in neighbor_lists]], dtype=np.float64), n, axis=0)
    if candidates.exact_cells:
        keys = np.array(list(candidates.exact_cells.keys()), dtype=np.int64)
        hi[keys[:, 0], keys[:, 1]] = np.fromiter(candidates.exact_cells.values(), dtype=np.float64,
                                                 count=len(keys))
    np.maximum(hi, lo, out=hi)
    return CellBounds(lo, hi)


def save_candidates(path, candidates: CandidateSet, neighbor_lists, bounds: CellBounds, *, k_prime: int,
                    similarity: Similarity, query_path: str | None = None,
                    manifest_path: str | None = None) -> None:
    """pipeline.py:188-213 — deterministic JSON artifact, written atomically."""
    payload = {
        "format": CANDIDATES_FORMAT,
        "k_prime": k_prime,
        "n_candidates": len(candidates),
        "n_query_tokens": len(neighbor_lists),
        "doc_ids": list(candidates.doc_ids),
        "doc_indices": list(candidates.doc_indices),
        "kth_sim": [nl.kth_similarity for nl in neighbor_lists],
        "exact_pairs": sorted([r, t] for (r, t) in candidates.exact_cells),
        "lo": float(bounds.lo[0, 0]),
        "hi": [[float(v) for v in row] for row in bounds.hi],
        "similarity": {"kind": similarity.kind, "range": [similarity.range_lo, similarity.range_hi],
                       "clamp_negative": similarity.clamp_negative},
        "query_path": query_path,
        "manifest_path": manifest_path,
    }
    target = Path(path)
    tmp = target.with_name(target.name + ".tmp")
    tmp.write_text(json.dumps(payload, sort_keys=True, indent=1) + "\n")
    tmp.replace(target)


def load_candidates(path) -> dict:
    """pipeline.py:216-230."""
    p = Path(path)
    payload = json.loads(p.read_text())
    if not isinstance(payload, dict) or payload.get("format") != CANDIDATES_FORMAT:
        raise ValueError(f"{p}: not a candidate artifact (format field mismatch)")
    required = ("k_prime", "doc_ids", "doc_indices", "kth_sim", "exact_pairs", "lo", "hi", "similarity")
    missing = [key for key in required if key not in payload]
    if missing:
        raise ValueError(f"{p}: candidate artifact missing fields {missing}")
    n, t = len(payload["doc_ids"]), len(payload["kth_sim"])
    hi = payload["hi"]
    if len(hi) != n or any(len(row) != t for row in hi):
        raise ValueError(f"{p}: hi bounds shape does not match {n} docs x {t} tokens")
    return payload
