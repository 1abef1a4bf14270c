"""Device-resident CSR batches and the batched P1 entry points.

A :class:`TokenBatch` is many ``MaxSimOracle(query, docs)`` instances
(colbandit/oracle.py:107-144) packed into five device arrays: query tokens,
query-token offsets, document tokens, document-token offsets and per-query
document ranges. Tokens stay in their storage dtype (fp16 / bf16 / fp32 /
fp64) — the reference's float64 upcast (validation.py:14) happens implicitly
inside the kernels, which accumulate exact products.

Entry points (all stream-ordered on torch's current stream):

* :func:`maxsim_scores`  — dense MaxSim score of every candidate (P1 kernel)
* :func:`rerank_topk`    — scores + per-query Top-K (the exhaustive reranker)
* :func:`exact_cells`    — float64-exact cell matrix + fsum row scores
* :func:`topk`           — per-query Top-K of a score vector
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib

__all__ = ["TokenBatch", "maxsim_scores", "rerank_topk", "exact_cells", "topk", "dtype_code"]

_PATHS = {"auto": _lib.CBX_PATH_AUTO, "tc": _lib.CBX_PATH_TC, "tcgen05": _lib.CBX_PATH_TC, "simt": _lib.CBX_PATH_SIMT}


def dtype_code(tdtype) -> int:
    import torch

    codes = {torch.float32: _lib.CBX_F32, torch.float16: _lib.CBX_F16, torch.bfloat16: _lib.CBX_BF16,
             torch.float64: _lib.CBX_F64}
    if tdtype not in codes:
        raise ValueError(f"unsupported token dtype {tdtype}; expected float16, bfloat16, float32 or float64")
    return codes[tdtype]


def to_torch_tokens(arr, dtype: str | None = None):
    """numpy / torch token matrix -> CPU torch tensor in its storage dtype.

    numpy uint16 arrays are bf16 bit patterns and need ``dtype="bf16"``.
    """
    import torch

    if isinstance(arr, torch.Tensor):
        return arr
    a = np.ascontiguousarray(arr)
    if dtype == "bf16" or (a.dtype == np.uint16 and dtype is None):
        if a.dtype != np.uint16:
            raise ValueError("bf16 tokens must be given as uint16 bit patterns or a torch.bfloat16 tensor")
        return torch.from_numpy(a.view(np.int16) if a.flags.writeable else a.view(np.int16).copy()).view(torch.bfloat16)
    if a.dtype not in (np.float16, np.float32, np.float64):
        a = a.astype(np.float64)
    if not a.flags.writeable:
        a = a.copy()
    return torch.from_numpy(a)


@dataclass
class TokenBatch:
    q_tokens: "object"    # torch [n_q_tokens, dim]
    q_tok_off: "object"   # torch int64 [n_queries + 1]
    d_tokens: "object"    # torch [n_d_tokens, dim]
    d_tok_off: "object"   # torch int64 [n_docs + 1]
    q_doc_off: "object"   # torch int64 [n_queries + 1]
    clamp_negative: bool = False
    max_lq: int = 0
    max_q_docs: int = 0
    max_q_doc_tokens: int = 0

    # -------------------------------------------------------------- construction
    @classmethod
    def from_device(cls, q_tokens, q_tok_off, d_tokens, d_tok_off, q_doc_off, clamp_negative=False,
                    host_offsets=None) -> "TokenBatch":
        """Wrap device tensors; host copies of the offsets (given or fetched) size the launch."""
        if host_offsets is None:
            host_offsets = (q_tok_off.cpu().numpy(), d_tok_off.cpu().numpy(), q_doc_off.cpu().numpy())
        qo, do, qd = (np.asarray(x, dtype=np.int64) for x in host_offsets)
        lq = np.diff(qo)
        ndocs = np.diff(qd)
        qtoks = do[qd[1:]] - do[qd[:-1]] if len(qd) > 1 else np.zeros(0, np.int64)
        b = cls(q_tokens, q_tok_off, d_tokens, d_tok_off, q_doc_off, bool(clamp_negative),
                int(lq.max()) if len(lq) else 0, int(ndocs.max()) if len(ndocs) else 0,
                int(qtoks.max()) if len(qtoks) else 0)
        b.host_offsets = (qo, do, qd)
        b._validate()
        return b

    @classmethod
    def from_host(cls, queries: Sequence, docs: Sequence[Sequence], dtype: str | None = None,
                  clamp_negative: bool = False, device=None) -> "TokenBatch":
        """Pack host queries and per-query doc lists (numpy or torch) into one device batch."""
        torch = _lib.require_cuda()
        if len(queries) != len(docs):
            raise ValueError("one candidate list per query is required")
        qt = [to_torch_tokens(q, dtype) for q in queries]
        dt = [[to_torch_tokens(d, dtype) for d in dl] for dl in docs]
        flat_docs = [d for dl in dt for d in dl]
        tdt = qt[0].dtype if qt else torch.float32
        for t in qt + flat_docs:
            if t.dtype != tdt:
                raise ValueError("all token matrices of a batch must share one dtype")
        qo = np.zeros(len(qt) + 1, np.int64)
        np.cumsum([t.shape[0] for t in qt], out=qo[1:])
        do = np.zeros(len(flat_docs) + 1, np.int64)
        np.cumsum([t.shape[0] for t in flat_docs], out=do[1:])
        qd = np.zeros(len(dt) + 1, np.int64)
        np.cumsum([len(dl) for dl in dt], out=qd[1:])
        device = device or torch.device("cuda", torch.cuda.current_device())
        dim = qt[0].shape[1] if qt else 1
        qcat = torch.cat(qt).contiguous() if qt else torch.zeros((0, dim), dtype=tdt)
        dcat = torch.cat(flat_docs).contiguous() if flat_docs else torch.zeros((0, dim), dtype=tdt)
        return cls.from_device(
            qcat.to(device, non_blocking=False), torch.from_numpy(qo).to(device), dcat.to(device),
            torch.from_numpy(do).to(device), torch.from_numpy(qd).to(device), clamp_negative,
            host_offsets=(qo, do, qd))

    def _validate(self) -> None:
        import torch

        for name in ("q_tokens", "d_tokens"):
            t = getattr(self, name)
            if not t.is_cuda:
                raise ValueError(f"{name} must live on a CUDA device")
            if t.dim() != 2:
                raise ValueError(f"{name} must be 2-D (tokens x dim)")
            if not t.is_contiguous():
                raise ValueError(f"{name} must be contiguous")
            if t.data_ptr() % 16:
                raise ValueError(f"{name} must be 16-byte aligned")
        if self.q_tokens.dtype != self.d_tokens.dtype:
            raise ValueError("query and document tokens must share one dtype")
        if self.q_tokens.shape[1] != self.d_tokens.shape[1]:
            raise ValueError(
                f"doc embedding dim {self.d_tokens.shape[1]} does not match query dim {self.q_tokens.shape[1]}")
        for name in ("q_tok_off", "d_tok_off", "q_doc_off"):
            t = getattr(self, name)
            if t.dtype != torch.int64 or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous int64 CUDA tensor")
        dtype_code(self.q_tokens.dtype)

    # -------------------------------------------------------------- properties
    @property
    def n_queries(self) -> int:
        return self.q_doc_off.shape[0] - 1

    @property
    def n_docs(self) -> int:
        return self.d_tok_off.shape[0] - 1

    @property
    def dim(self) -> int:
        return int(self.q_tokens.shape[1])

    def struct(self) -> _lib.CbxBatch:
        s = _lib.CbxBatch()
        s.q_tokens = self.q_tokens.data_ptr()
        s.q_tok_off = self.q_tok_off.data_ptr()
        s.d_tokens = self.d_tokens.data_ptr()
        s.d_tok_off = self.d_tok_off.data_ptr()
        s.q_doc_off = self.q_doc_off.data_ptr()
        s.n_queries = self.n_queries
        s.n_docs = self.n_docs
        s.n_q_tokens = int(self.q_tokens.shape[0])
        s.n_d_tokens = int(self.d_tokens.shape[0])
        s.dim = self.dim
        s.dtype = dtype_code(self.q_tokens.dtype)
        s.clamp_negative = 1 if self.clamp_negative else 0
        s.max_lq = self.max_lq
        s.max_q_docs = self.max_q_docs
        s.max_q_doc_tokens = self.max_q_doc_tokens
        s.d_norm_max = getattr(self, "_norm_max", 0.0) or 0.0
        return s

    def norm_max(self) -> float:
        """Upper bound on every document token's L2 norm (one device pass, cached): the bandit's fp32
        reveal screen bounds its rounding error with it (cbx_batch.d_norm_max)."""
        v = getattr(self, "_norm_max", None)
        if v is None:
            import torch

            out = torch.zeros(1, dtype=torch.float32, device=self.d_tokens.device)
            if self.d_tokens.shape[0]:
                _lib.check(_lib.load().cbx_token_norm_max(self.d_tokens.data_ptr(), int(self.d_tokens.shape[0]),
                                                          self.dim, dtype_code(self.d_tokens.dtype), out.data_ptr(),
                                                          _stream_ptr()), "token_norm_max")
            v = float(out.item())
            # an all-zero (or empty) token set still needs a positive bound for the C ABI
            v = v if v > 0.0 else 1e-30
            self._norm_max = v
        return v


def _stream_ptr():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _workspace(nbytes: int):
    import torch

    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device="cuda")


def maxsim_scores(batch: TokenBatch, path: str = "auto", out=None):
    """float32 MaxSim score of every candidate document of the batch."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    if path not in _PATHS:
        raise ValueError(f"path must be one of {sorted(_PATHS)}, got {path!r}")
    if out is None:
        out = torch.empty(batch.n_docs, dtype=torch.float32, device=batch.d_tokens.device)
    s = batch.struct()
    _lib.check(lib.cbx_maxsim_scores(ctypes.byref(s), out.data_ptr(), _PATHS[path], None, 0, _stream_ptr()),
               "maxsim_scores")
    return out


def topk(scores, q_doc_off, k: int, max_q_docs: int):
    """Per-query Top-K (query-local indices, values) of float32 or float64 scores."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    nq = q_doc_off.shape[0] - 1
    if k < 0:
        raise ValueError(f"k must be non-negative, got {k}")
    idx = torch.empty((nq, k), dtype=torch.int32, device=scores.device)
    val = torch.empty((nq, k), dtype=scores.dtype, device=scores.device)
    s = _lib.CbxBatch()
    s.n_queries, s.max_q_docs = nq, max_q_docs
    ws = _workspace(lib.cbx_workspace_bytes(ctypes.byref(s), k))
    fn = lib.cbx_topk_f32 if scores.dtype == torch.float32 else lib.cbx_topk_f64
    _lib.check(fn(scores.data_ptr(), q_doc_off.data_ptr(), nq, max_q_docs, k, idx.data_ptr(), val.data_ptr(),
                  ws.data_ptr(), ws.numel(), _stream_ptr()), "topk")
    return idx, val


def rerank_topk(batch: TokenBatch, k: int, path: str = "auto"):
    """Exhaustive reranking: (Top-K local indices [nq, k], Top-K scores, all scores)."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    if path not in _PATHS:
        raise ValueError(f"path must be one of {sorted(_PATHS)}, got {path!r}")
    nq = batch.n_queries
    scores = torch.empty(batch.n_docs, dtype=torch.float32, device=batch.d_tokens.device)
    idx = torch.empty((nq, k), dtype=torch.int32, device=scores.device)
    val = torch.empty((nq, k), dtype=torch.float32, device=scores.device)
    s = batch.struct()
    ws = _workspace(lib.cbx_workspace_bytes(ctypes.byref(s), k))
    _lib.check(lib.cbx_rerank_topk(ctypes.byref(s), k, _PATHS[path], scores.data_ptr(), idx.data_ptr(),
                                   val.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr()), "rerank_topk")
    return idx, val, scores


def exact_cells(batch: TokenBatch, with_scores: bool = True):
    """float64-exact cells [n_docs, max_lq] (NaN beyond each query's Lq) and fsum row scores."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    ld = max(batch.max_lq, 1)
    cells = torch.full((batch.n_docs, ld), float("nan"), dtype=torch.float64, device=batch.d_tokens.device)
    scores = torch.empty(batch.n_docs, dtype=torch.float64, device=cells.device) if with_scores else None
    s = batch.struct()
    _lib.check(lib.cbx_maxsim_cells_f64(ctypes.byref(s), cells.data_ptr(), ld,
                                        scores.data_ptr() if scores is not None else None, _stream_ptr()),
               "exact_cells")
    return cells, scores


class HostBatch:
    """A TokenBatch's arrays in pinned host memory plus reusable device buffers.

    ``rerank_topk_host`` is the end-to-end public call: host->device copies of
    the step's inputs, the exhaustive reranker, device->host copy of the
    per-query Top-K — all stream-ordered on one stream.
    """

    def __init__(self, q_tokens, q_tok_off, d_tokens, d_tok_off, q_doc_off, clamp_negative=False):
        torch = _lib.require_cuda()
        pin = lambda t: t.contiguous().pin_memory()  # noqa: E731
        self.host = [pin(t) for t in (q_tokens, q_tok_off, d_tokens, d_tok_off, q_doc_off)]
        self.dev = [torch.empty_like(t, device="cuda") for t in self.host]
        self.clamp_negative = clamp_negative
        offs = [t.numpy() for t in self.host[1::2]]
        self.batch = TokenBatch.from_device(*self.dev, clamp_negative=clamp_negative,
                                            host_offsets=(offs[0], offs[1], self.host[4].numpy()))

    @classmethod
    def from_device_batch(cls, b: TokenBatch) -> "HostBatch":
        return cls(b.q_tokens.cpu(), b.q_tok_off.cpu(), b.d_tokens.cpu(), b.d_tok_off.cpu(), b.q_doc_off.cpu(),
                   b.clamp_negative)

    @property
    def h2d_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.host)


def rerank_topk_host(hb: HostBatch, k: int, path: str = "auto", out=None):
    """End-to-end exhaustive reranking from pinned host buffers to host Top-K."""
    torch = _lib.require_cuda()
    for h, d in zip(hb.host, hb.dev):
        d.copy_(h, non_blocking=True)
    idx, val, _ = rerank_topk(hb.batch, k, path)
    if out is None:
        out = (torch.empty(idx.shape, dtype=idx.dtype).pin_memory(),
               torch.empty(val.shape, dtype=val.dtype).pin_memory())
    out[0].copy_(idx, non_blocking=True)
    out[1].copy_(val, non_blocking=True)
    return out


class Corpus:
    """An HBM-resident document collection scored against per-call candidate lists.

    The reranking-service form of the reference's ``ColBanditReranker``:
    ``fit`` stores the corpus once (reranker.py:86-104), every ``rerank``
    scores one candidate pool per query (reranker.py:115-141). Here the
    corpus tokens live in HBM; a call ships only query tokens and candidate
    ids host -> device, packs the candidates with ``cbx_gather_candidates``
    and runs the exhaustive reranker, returning the per-query Top-K
    (positions in each query's candidate list) to the host.
    """

    def __init__(self, doc_tokens, doc_offsets, dtype: str | None = None, clamp_negative: bool = False):
        torch = _lib.require_cuda()
        off = np.ascontiguousarray(np.asarray(doc_offsets, dtype=np.int64))
        if off.ndim != 1 or len(off) < 2 or off[0] != 0 or np.any(np.diff(off) <= 0):
            raise ValueError("doc_offsets must start at 0 and grow strictly (every document needs a token)")
        if isinstance(doc_tokens, torch.Tensor) and doc_tokens.is_cuda:
            self.tokens = doc_tokens.contiguous()
        else:
            self.tokens = to_torch_tokens(doc_tokens, dtype).contiguous().cuda()
        if self.tokens.dim() != 2 or self.tokens.shape[0] != off[-1]:
            raise ValueError("doc_tokens must be [doc_offsets[-1], dim]")
        dtype_code(self.tokens.dtype)
        self.offsets_host = off
        self.lengths = np.diff(off)
        self.offsets = torch.from_numpy(off).cuda()
        self.clamp_negative = bool(clamp_negative)
        self.doc_ids = None
        self._ws = {}
        self._norm_max = None

    @classmethod
    def from_docs(cls, docs, clamp_negative: bool = False) -> "Corpus":
        """Upload a list of DocTokens (or token matrices) once; mixed dtypes widen to the widest one."""
        import torch

        from .oracle import DocTokens

        stores = [d._store if isinstance(d, DocTokens) else to_torch_tokens(d) for d in docs]
        if not stores:
            raise ValueError("corpus must contain at least one document")
        dts = {t.dtype for t in stores}
        if len(dts) > 1:
            order = [torch.float16, torch.bfloat16, torch.float32, torch.float64]
            wide = max(dts, key=order.index)
            if dts == {torch.float16, torch.bfloat16}:
                wide = torch.float32
            stores = [t.to(wide) for t in stores]
        off = np.zeros(len(stores) + 1, np.int64)
        np.cumsum([t.shape[0] for t in stores], out=off[1:])
        c = cls(torch.cat([t.cpu() for t in stores]).contiguous(), off, clamp_negative=clamp_negative)
        c.doc_ids = [d.doc_id if isinstance(d, DocTokens) else f"doc{i:04d}" for i, d in enumerate(docs)]
        return c

    @property
    def n_tokens(self) -> int:
        return int(self.tokens.shape[0])

    def widened(self, dtype) -> "Corpus":
        """A cached copy of this corpus in a wider dtype (for queries the storage dtype cannot hold exactly)."""
        key = ("wide", dtype)
        c = self._ws.get(key)
        if c is None:
            c = Corpus(self.tokens.to(dtype), self.offsets_host, clamp_negative=self.clamp_negative)
            c.doc_ids = self.doc_ids
            self._ws[key] = c
        return c

    def norm_max(self) -> float:
        """Largest token L2 norm (device reduction, computed once; bounds the tcgen05 Stage-1 error)."""
        if self._norm_max is None:
            import torch

            out = torch.zeros(1, dtype=torch.float32, device=self.tokens.device)
            lib = _lib.load()
            _lib.check(lib.cbx_token_norm_max(self.tokens.data_ptr(), self.n_tokens, self.dim,
                                              dtype_code(self.tokens.dtype), out.data_ptr(),
                                              ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
                       "token_norm_max")
            self._norm_max = float(out.item())
        return self._norm_max

    def gather(self, cand_ids):
        """Pack corpus documents ``cand_ids`` (int64, host) into contiguous device rows + CSR offsets."""
        import torch

        lib = _lib.load()
        cid = np.ascontiguousarray(np.asarray(cand_ids, dtype=np.int64))
        if len(cid) and (cid.min() < 0 or cid.max() >= self.n_docs):
            raise IndexError(f"candidate id out of range [0, {self.n_docs})")
        total = int(self.lengths[cid].sum()) if len(cid) else 0
        rows = torch.empty((max(total, 1), self.dim), dtype=self.tokens.dtype, device=self.tokens.device)[:total]
        doff = torch.zeros(len(cid) + 1, dtype=torch.int64, device=self.tokens.device)
        status = torch.zeros(1, dtype=torch.int32, device=self.tokens.device)
        dcid = torch.from_numpy(cid).to(self.tokens.device)
        _lib.check(lib.cbx_gather_candidates(self.tokens.data_ptr(), self.offsets.data_ptr(), self.n_docs, self.dim,
                                             dtype_code(self.tokens.dtype), dcid.data_ptr(), len(cid),
                                             rows.data_ptr(), total, doff.data_ptr(), status.data_ptr(),
                                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "gather")
        host_off = np.zeros(len(cid) + 1, np.int64)
        if len(cid):
            np.cumsum(self.lengths[cid], out=host_off[1:])
        return rows, doff, host_off

    @property
    def n_docs(self) -> int:
        return len(self.lengths)

    @property
    def dim(self) -> int:
        return int(self.tokens.shape[1])

    def _buf(self, name, numel, dtype, pinned=False):
        import torch

        t = self._ws.get(name)
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = torch.empty(max(int(numel), 1), dtype=dtype, pin_memory=pinned) if pinned else \
                torch.empty(max(int(numel), 1), dtype=dtype, device="cuda")
            self._ws[name] = t
        return t[:numel]

    def rerank_topk(self, q_tokens, q_tok_off, cand_ids, q_cand_off, k: int, path: str = "auto", sync: bool = True,
                    mode: str = "packed"):
        """Host in, host out: per-query Top-K positions into the candidate list and their scores.

        ``q_tokens`` [sum Lq, dim] (pinned CPU tensor in the corpus dtype), ``q_tok_off`` [nq + 1],
        ``cand_ids`` [sum N_q] corpus document ids, ``q_cand_off`` [nq + 1] (int64 numpy or CPU tensors).
        ``mode="packed"`` streams the candidates straight from the corpus (tcgen05 path, no copy);
        ``mode="gather"`` first packs them into a contiguous batch (any dtype / path).
        ``sync=False`` returns at once: the returned pinned tensors are the call's own (later calls never
        overwrite them) and become valid when the stream reaches them; a bad candidate id is reported by
        ``synchronize()`` or by the next call.
        """
        import torch

        lib = _lib.load()
        qo = np.asarray(q_tok_off, dtype=np.int64)
        co = np.asarray(q_cand_off, dtype=np.int64)
        cid = cand_ids if isinstance(cand_ids, torch.Tensor) else torch.from_numpy(np.asarray(cand_ids, np.int64))
        nq = len(qo) - 1
        n_cand = int(co[-1])
        if cid.numel() != n_cand:
            raise ValueError("cand_ids length does not match q_cand_off[-1]")
        cid_np = cid.numpy()
        if mode not in ("packed", "gather"):
            raise ValueError(f"mode must be 'packed' or 'gather', got {mode!r}")
        # packed mode checks the ids on the device (a bad id scores as an empty document and raises
        # IndexError at the synchronisation below); the gather mode sizes its copy on the host
        if mode == "gather" and n_cand and (cid_np.min() < 0 or cid_np.max() >= self.n_docs):
            raise IndexError(f"candidate id out of range [0, {self.n_docs})")
        # an asynchronous call (sync=False) must not share pinned staging with a call still in flight: it
        # takes fresh blocks from torch's caching host allocator (which holds a block until the copies that
        # used it have completed) and its status is checked at the next synchronisation
        self._check_pending(wait=sync)
        pinned = (lambda name, n, dt: self._buf(name, n, dt, pinned=True)) if sync else \
            (lambda name, n, dt: torch.empty(max(int(n), 1), dtype=dt, pin_memory=True)[:n])
        # host -> device: the call's inputs only
        dq = self._buf("q", q_tokens.numel(), q_tokens.dtype).view(q_tokens.shape)
        dq.copy_(q_tokens, non_blocking=True)
        hoff = pinned("hoff", 2 * (nq + 1), torch.int64)
        hoff[: nq + 1].copy_(torch.from_numpy(qo))
        hoff[nq + 1:].copy_(torch.from_numpy(co))
        doffs = self._buf("offs", 2 * (nq + 1), torch.int64)
        doffs.copy_(hoff, non_blocking=True)
        dqo, dco = doffs[: nq + 1], doffs[nq + 1:]
        dcid = self._buf("cid", n_cand, torch.int64)
        dcid.copy_(cid, non_blocking=True)
        status = self._buf("status", 1, torch.int32)
        status.zero_()
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        nd = np.diff(co)
        max_lq = int(np.diff(qo).max()) if nq else 0
        max_nc = int(nd.max()) if nq else 0
        if mode == "packed":
            s_ = _lib.CbxBatch()
            s_.q_tokens, s_.q_tok_off = dq.data_ptr(), dqo.data_ptr()
            s_.d_tokens, s_.d_tok_off, s_.q_doc_off = self.tokens.data_ptr(), self.offsets.data_ptr(), dco.data_ptr()
            s_.n_queries, s_.n_docs = nq, n_cand
            s_.n_q_tokens, s_.n_d_tokens = int(dq.shape[0]), int(self.tokens.shape[0])
            s_.dim, s_.dtype = self.dim, dtype_code(self.tokens.dtype)
            s_.clamp_negative, s_.max_lq, s_.max_q_docs, s_.max_q_doc_tokens = int(self.clamp_negative), max_lq, max_nc, 0
            ws = self._buf("ws", lib.cbx_corpus_workspace_bytes(nq, n_cand, max_nc, k), torch.uint8)
            scores = self._buf("scores", n_cand, torch.float32)
            idx = self._buf("idx", nq * k, torch.int32).view(nq, k)
            val = self._buf("val", nq * k, torch.float32).view(nq, k)
            _lib.check(lib.cbx_corpus_rerank_topk(ctypes.byref(s_), self.offsets.data_ptr(), self.n_docs,
                                                  dcid.data_ptr(), k, scores.data_ptr(), idx.data_ptr(),
                                                  val.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(),
                                                  stream), "corpus_rerank_topk")
        else:
            total_rows = int(self.lengths[cid_np].sum()) if n_cand else 0
            rows = self._buf("rows", total_rows * self.dim, self.tokens.dtype).view(total_rows, self.dim)
            doff = self._buf("doff", n_cand + 1, torch.int64)
            _lib.check(lib.cbx_gather_candidates(self.tokens.data_ptr(), self.offsets.data_ptr(), self.n_docs,
                                                 self.dim, dtype_code(self.tokens.dtype), dcid.data_ptr(), n_cand,
                                                 rows.data_ptr(), total_rows, doff.data_ptr(), status.data_ptr(),
                                                 stream), "gather")
            b = TokenBatch(dq, dqo, rows, doff, dco, self.clamp_negative, max_lq, max_nc, total_rows)
            idx, val, _ = rerank_topk(b, k, path)
        out_i = pinned("oi", idx.numel(), torch.int32).view(idx.shape)
        out_v = pinned("ov", val.numel(), torch.float32).view(val.shape)
        out_i.copy_(idx, non_blocking=True)
        out_v.copy_(val, non_blocking=True)
        st_h = pinned("st_h", 1, torch.int32)
        st_h.copy_(status, non_blocking=True)  # read back with the outputs: one synchronisation per call
        if sync:
            torch.cuda.current_stream().synchronize()
            if int(st_h[0]):
                raise IndexError("candidate id out of range")
        else:
            ev = torch.cuda.Event()
            ev.record()
            self._pending.append((ev, st_h))
        return out_i, out_v

    def _check_pending(self, wait: bool):
        """Status of earlier sync=False calls: completed ones are checked (all of them when ``wait``)."""
        pend = getattr(self, "_pending", None)
        if pend is None:
            pend = self._pending = []
        keep = []
        bad = False
        for ev, st_h in pend:
            if wait:
                ev.synchronize()
            elif not ev.query():
                keep.append((ev, st_h))
                continue
            bad |= bool(int(st_h[0]))
        self._pending = keep
        if bad:
            raise IndexError("candidate id out of range (in an earlier rerank_topk(sync=False) call)")

    def synchronize(self):
        """Wait for every rerank_topk(sync=False) call in flight; raises IndexError if one saw a bad candidate id."""
        self._check_pending(wait=True)
