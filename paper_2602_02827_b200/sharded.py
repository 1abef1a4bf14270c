"""Document-sharded Col-Bandit: one query over a candidate pool split across GPUs.

SURVEY §8(e), BASELINE cfg4 at 2/4/8 GPUs. Rank r holds the token embeddings
of a contiguous document range only (``dist.balanced_ranges``) but keeps the
whole compact run state — per-row Welford statistics, exact sums, intervals,
the four selection trees and the PCG64 stream, ~100 B per row — and takes
every decision itself. Because all ranks start from the same state and draw
the same numbers, they agree on every stop test, boundary pair (i+, i-),
selected row i* and column t* (colbandit/bandit.py:249-327) without talking;
only the owner of i* can compute the cell, so each iteration exchanges
exactly one value: ``cbx_bandit_shard_step`` writes the owner's ordered key
(and INT64_MIN on every other rank) and one all-reduce MAX of 8 bytes hands
it to all ranks, which then apply the identical update (bandit.py:220-247).
The lazy warm-up (one cell per row, bandit.py:285-296) is computed where the
rows live and exchanged once as an N-slot all-reduce. The result is
reveal-for-reveal the single-GPU trace on every rank.

Two exchange paths implement the same protocol:

* ``ShardedBanditRun`` + ``drive``: a host-launched step kernel per iteration
  and a collective (NCCL all-reduce over NVLink on the box, gloo in CPU tests)
  — bounded by kernel-launch + collective latency;
* ``MailboxRun`` (``run_mailbox`` across processes, ``run_local_shards`` for
  several ranks in one launch): ONE persistent kernel per rank for the whole
  run (``cbx_bandit_shard_run``). The owner of a revealed cell stores it into
  every other rank's inbox over NVLink peer memory (CUDA IPC mappings; value,
  then a system-scope release store of a flag) and the others spin on their
  own inbox — the per-iteration exchange costs one NVLink store latency
  instead of a launch plus a collective.

The path exists for pools whose embeddings do not fit one GPU (DESIGN.md §7
gives the measured numbers).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .bandit import _MODE_CODE, MAX_COLS, TREE_ROWS, BanditConfig, Reveals, RunResult, _rng_state
from .bounds import CellBounds

__all__ = ["ShardedBanditRun", "drive", "allreduce_exchange", "shard_batch", "xchg_key", "xchg_value",
           "NOT_MINE", "MailboxRun", "run_mailbox", "run_local_shards"]

NOT_MINE = -(1 << 63)  # INT64_MIN: the slot value of a rank that does not own the cell


def xchg_key(v: float) -> int:
    """Host mirror of the kernel's exchange encoding: float64 -> int64 whose signed order is the value order."""
    u = int(np.float64(v).view(np.uint64))
    k = (~u & (2 ** 64 - 1)) if u >> 63 else (u | (1 << 63))
    k ^= 1 << 63
    return k - (1 << 64) if k >> 63 else k


def xchg_value(k: int) -> float:
    """Inverse of ``xchg_key``."""
    u = (k + (1 << 64)) % (1 << 64) ^ (1 << 63)
    u = (u & ((1 << 63) - 1)) if u >> 63 else (~u & (2 ** 64 - 1))
    return float(np.uint64(u).view(np.float64))


def shard_batch(query, doc_tokens, doc_offsets, own: tuple[int, int], clamp_negative: bool = False):
    """A TokenBatch for one rank: the query, and the tokens of documents own[0]:own[1] of a pool whose
    CSR offsets (all documents) are ``doc_offsets``; other documents are present as empty rows.

    ``doc_tokens`` holds the rank's tokens only: rows doc_offsets[own[0]]:doc_offsets[own[1]] of the pool.
    """
    import torch

    from .batch import TokenBatch, to_torch_tokens

    torch_ = _lib.require_cuda()
    off = np.asarray(doc_offsets, dtype=np.int64)
    lo, hi = int(own[0]), int(own[1])
    n = len(off) - 1
    if not 0 <= lo <= hi <= n:
        raise ValueError(f"owned range {own} outside the pool of {n} documents")
    base = off[lo]
    local = np.zeros(n + 1, np.int64)
    local[lo:hi + 1] = off[lo:hi + 1] - base
    local[hi + 1:] = off[hi] - base
    dev = torch_.device("cuda", torch_.cuda.current_device())
    q = to_torch_tokens(query).to(dev).contiguous()
    d = to_torch_tokens(doc_tokens).to(dev).contiguous()
    if d.shape[0] != int(off[hi] - base):
        raise ValueError(f"rank holds {d.shape[0]} tokens, its documents have {int(off[hi] - base)}")
    qo = np.array([0, q.shape[0]], np.int64)
    qd = np.array([0, n], np.int64)
    return TokenBatch.from_device(q, torch.from_numpy(qo).to(dev), d, torch.from_numpy(local).to(dev),
                                  torch.from_numpy(qd).to(dev), clamp_negative, host_offsets=(qo, local, qd))


class ShardedBanditRun:
    """One rank's share of a document-sharded run: device state, exchange slots, outputs."""

    def __init__(self, batch, own: tuple[int, int], cfg: BanditConfig,
                 bounds: CellBounds | tuple[float, float] = (-1.0, 1.0), selection: str = "auto"):
        torch = _lib.require_cuda()
        self._lib = _lib.load()
        N, T = batch.n_docs, int(batch.q_tokens.shape[0])
        if T > MAX_COLS:
            raise ValueError(f"the device bandit supports at most {MAX_COLS} query tokens, got {T}")
        if not 1 <= cfg.k <= N:
            raise ValueError(f"k={cfg.k} must be in [1, {N}] for a sharded run")
        self.batch, self.cfg, self.n_rows, self.n_cols = batch, cfg, N, T
        self.own = (int(own[0]), int(own[1]))
        d = _lib.CbxBanditRunDesc()
        d.query, d.row_begin, d.n_rows, d.n_cols, d.k = 0, 0, N, T, cfg.k
        d.explore_mode = _MODE_CODE[cfg.explore_mode]
        d.alpha_ef, d.epsilon = cfg.alpha_ef, cfg.epsilon
        d.log_term = cfg.radius_config.log_term(N, T)
        uni = bounds if isinstance(bounds, tuple) else bounds.uniform_values()
        dev = torch.device("cuda", torch.cuda.current_device())
        self._lo = self._hi = None
        if uni:
            d.bounds_off = -1
            d.lo_uniform, d.hi_uniform = uni
        else:
            d.bounds_off = 0
            self._lo = torch.from_numpy(np.ascontiguousarray(bounds.lo, dtype=np.float64).ravel()).to(dev)
            self._hi = torch.from_numpy(np.ascontiguousarray(bounds.hi, dtype=np.float64).ravel()).to(dev)
        d.rng, warm = _rng_state(cfg.seed, cfg.explore_mode, cfg.gamma_init, N * T)
        d.n_warm, d.warm_off = len(warm), 0
        tree = selection == "tree" or (selection == "auto" and N > TREE_ROWS)
        d.flags = _lib.CBX_BANDIT_TREE if tree else 0
        d.trace_off, d.state_off = 0, 0
        self._desc_host = d
        self.warm_slots = N if cfg.explore_mode == "epsilon-greedy" else len(warm)
        self._desc = torch.frombuffer(bytearray(bytes(d)), dtype=torch.uint8).to(dev)
        self._warm = torch.from_numpy(warm).to(dev) if len(warm) else None
        self._state_bytes = self._lib.cbx_bandit_state_bytes(N + _lib.CBX_BANDIT_ROW_SLACK)
        self._state = torch.empty(self._state_bytes, dtype=torch.uint8, device=dev)
        self._step = torch.zeros(_lib.CBX_BANDIT_STEP_BYTES, dtype=torch.uint8, device=dev)
        self.xchg = torch.empty(max(N, len(warm), 1), dtype=torch.int64, device=dev)
        self._topk = torch.empty(cfg.k, dtype=torch.int32, device=dev)
        self._tr_i = torch.empty(N * T, dtype=torch.int32, device=dev)
        self._tr_t = torch.empty(N * T, dtype=torch.int32, device=dev)
        self._tr_v = torch.empty(N * T, dtype=torch.float64, device=dev)
        self._out = torch.empty(ctypes.sizeof(_lib.CbxBanditOut), dtype=torch.uint8, device=dev)
        self._phase_host = torch.empty(1, dtype=torch.int32, pin_memory=True)
        batch.norm_max()
        self._bstruct = batch.struct()
        self._first = 1
        self.steps = 0

    def step(self) -> None:
        """Apply the last exchange, decide, reveal what this rank owns (stream-ordered, no host sync)."""
        torch = _lib.require_cuda()
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        _lib.check(self._lib.cbx_bandit_shard_step(
            ctypes.byref(self._bstruct), None, 0, self._desc.data_ptr(), self.own[0], self.own[1], self._first,
            ptr(self._lo), ptr(self._hi), ptr(self._warm), self._state.data_ptr(), self._state_bytes,
            self._step.data_ptr(), self.xchg.data_ptr(), self._topk.data_ptr(), self.cfg.k, self._tr_i.data_ptr(),
            self._tr_t.data_ptr(), self._tr_v.data_ptr(), self._out.data_ptr(), stream), "bandit_shard_step")
        self._first = 0
        self.steps += 1

    def phase(self) -> int:
        """What the last step left to exchange (synchronises with the stream)."""
        import torch

        self._phase_host.copy_(self._step[:4].view(torch.int32))
        torch.cuda.current_stream().synchronize()
        return int(self._phase_host[0])

    def slots(self, phase: int) -> int:
        return self.warm_slots if phase == _lib.CBX_SHARD_WARMUP else 1

    def result(self) -> RunResult:
        out = np.frombuffer(self._out.cpu().numpy().tobytes(), dtype=np.dtype(
            [("n_reveals", "<i8"), ("iterations", "<i4"), ("terminated_by", "<i4"), ("status", "<i4"),
             ("pad", "<i4")]))[0]
        if out["status"] == 1:
            raise RuntimeError("internal error: both boundary rows exhausted while unseparated")
        if out["status"] != 0:
            raise RuntimeError(f"bandit kernel status {int(out['status'])} (exact-sum capacity exceeded)")
        n = int(out["n_reveals"])
        reveals = Reveals(self._tr_i[:n].cpu().numpy(), self._tr_t[:n].cpu().numpy(), self._tr_v[:n].cpu().numpy())
        term = "separation" if out["terminated_by"] == _lib.CBX_TERM_SEPARATION else "exhaustion"
        return RunResult([int(x) for x in self._topk.cpu().tolist()], n / (self.n_rows * self.n_cols), reveals,
                         int(out["iterations"]), term)


def allreduce_exchange(group=None):
    """Exchange = all-reduce MAX of the first n slots over the process group (NCCL or gloo)."""
    import torch.distributed as dist

    def exchange(xchg, n: int) -> None:
        dist.all_reduce(xchg[:n], op=dist.ReduceOp.MAX, group=group)

    return exchange


def drive(run, exchange, check_every: int = 64, graph: bool | None = None):
    """Run a sharded bandit to its stop rule: step, exchange, repeat.

    ``run`` needs step() / phase() / slots() / xchg / result(); ``exchange(xchg, n)`` must leave every rank
    with the element-wise MAX of the ranks' first n slots. Every rank reaches DONE at the same step (the
    state is replicated), so ranks issue identical collective sequences. Reveal exchanges are issued
    ``check_every`` at a time between host synchronisations — as one CUDA graph of ``check_every``
    (collective, step) pairs when the slots live on the GPU (``graph`` None = auto) — and steps after DONE
    return at once, their exchanges carrying nothing.
    """
    run.step()
    ph = run.phase()
    if ph == _lib.CBX_SHARD_WARMUP:
        exchange(run.xchg, run.slots(ph))
        run.step()
        ph = run.phase()
    if graph is None:
        graph = bool(getattr(run.xchg, "is_cuda", False))
    g = None
    while ph != _lib.CBX_SHARD_DONE:
        if ph != _lib.CBX_SHARD_REVEAL:
            raise RuntimeError(f"unexpected exchange phase {ph}")
        if graph:
            if g is None:
                import torch

                g = torch.cuda.CUDAGraph()
                torch.cuda.synchronize()
                with torch.cuda.graph(g):
                    for _ in range(check_every):
                        exchange(run.xchg, 1)
                        run.step()
                run.steps -= check_every  # captured, not executed
            g.replay()
            run.steps += check_every
        else:
            for _ in range(check_every):
                exchange(run.xchg, 1)
                run.step()
        ph = run.phase()
    return run.result()


class MailboxRun:
    """``n_local`` ranks of a document-sharded run as CTAs of ONE persistent launch (cbx_bandit_shard_run).

    ``owns`` lists each local rank's owned row range; ``rank0`` is the global rank of the first local one and
    ``n_ranks`` the run's world size. ``batch`` indexes rows globally (a shard_batch of the rank's tokens, or
    the whole pool when the local ranks share one GPU's copy). Inboxes are set with ``set_peers``.
    """

    def __init__(self, batch, owns, cfg: BanditConfig, bounds: CellBounds | tuple[float, float] = (-1.0, 1.0),
                 rank0: int = 0, n_ranks: int | None = None):
        torch = _lib.require_cuda()
        self._lib = _lib.load()
        N, T = batch.n_docs, int(batch.q_tokens.shape[0])
        if T > MAX_COLS:
            raise ValueError(f"the device bandit supports at most {MAX_COLS} query tokens, got {T}")
        if not 1 <= cfg.k <= N:
            raise ValueError(f"k={cfg.k} must be in [1, {N}] for a sharded run")
        self.batch, self.cfg, self.n_rows, self.n_cols = batch, cfg, N, T
        self.n_local = len(owns)
        self.rank0 = int(rank0)
        self.n_ranks = int(n_ranks if n_ranks is not None else self.n_local)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        d = _lib.CbxBanditRunDesc()
        d.query, d.row_begin, d.n_rows, d.n_cols, d.k = 0, 0, N, T, cfg.k
        d.explore_mode = _MODE_CODE[cfg.explore_mode]
        d.alpha_ef, d.epsilon = cfg.alpha_ef, cfg.epsilon
        d.log_term = cfg.radius_config.log_term(N, T)
        uni = bounds if isinstance(bounds, tuple) else bounds.uniform_values()
        self._lo = self._hi = None
        if uni:
            d.bounds_off = -1
            d.lo_uniform, d.hi_uniform = uni
        else:
            d.bounds_off = 0
            self._lo = torch.from_numpy(np.ascontiguousarray(bounds.lo, dtype=np.float64).ravel()).to(dev)
            self._hi = torch.from_numpy(np.ascontiguousarray(bounds.hi, dtype=np.float64).ravel()).to(dev)
        d.rng, warm = _rng_state(cfg.seed, cfg.explore_mode, cfg.gamma_init, N * T)
        d.n_warm, d.warm_off = len(warm), 0
        d.flags = _lib.CBX_BANDIT_TREE if N > TREE_ROWS else 0
        descs = []
        for c in range(self.n_local):
            d.trace_off, d.state_off = c * N * T, c * (N + _lib.CBX_BANDIT_ROW_SLACK)
            descs.append(bytes(d))
        self._desc = torch.frombuffer(bytearray(b"".join(descs)), dtype=torch.uint8).to(dev)
        own = np.array([[int(a), int(b)] for a, b in owns], dtype=np.int64).reshape(-1)
        self._own = torch.from_numpy(own).to(dev)
        self._warm = torch.from_numpy(warm).to(dev) if len(warm) else None
        self._state_bytes = self._lib.cbx_bandit_state_bytes(self.n_local * (N + _lib.CBX_BANDIT_ROW_SLACK))
        self._state = torch.empty(self._state_bytes, dtype=torch.uint8, device=dev)
        self._topk = torch.empty((self.n_local, cfg.k), dtype=torch.int32, device=dev)
        self._tr_i = torch.empty(self.n_local * N * T, dtype=torch.int32, device=dev)
        self._tr_t = torch.empty(self.n_local * N * T, dtype=torch.int32, device=dev)
        self._tr_v = torch.empty(self.n_local * N * T, dtype=torch.float64, device=dev)
        self._out = torch.empty(self.n_local * ctypes.sizeof(_lib.CbxBanditOut), dtype=torch.uint8, device=dev)
        batch.norm_max()
        self._bstruct = batch.struct()
        self._peers = None

    @property
    def slots(self) -> int:
        return self.n_rows * self.n_cols

    def set_peers(self, table) -> None:
        """``table[c][p]``: rank p's inbox (val, flag) device addresses as local rank c sees them."""
        import torch

        flat = (_lib.CbxMboxPeer * (self.n_local * self.n_ranks))()
        for c in range(self.n_local):
            for p in range(self.n_ranks):
                flat[c * self.n_ranks + p] = _lib.CbxMboxPeer(*table[c][p])
        self._peers = torch.frombuffer(bytearray(bytes(flat)), dtype=torch.uint8).to(self.dev)

    def launch(self) -> None:
        """Issue the persistent launch on the current stream (inboxes must be cleared and peers set)."""
        torch = _lib.require_cuda()
        if self._peers is None:
            raise RuntimeError("set_peers() first")
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(self._lib.cbx_bandit_shard_run(
            ctypes.byref(self._bstruct), None, 0, self._desc.data_ptr(), self.n_local, self._own.data_ptr(),
            self.rank0, self.n_ranks, self._peers.data_ptr(), self.n_rows, ptr(self._lo), ptr(self._hi),
            ptr(self._warm), self._state.data_ptr(), self._state_bytes, self._topk.data_ptr(), self.cfg.k,
            self._tr_i.data_ptr(), self._tr_t.data_ptr(), self._tr_v.data_ptr(), self._out.data_ptr(), stream),
            "bandit_shard_run")

    def results(self) -> list:
        out = np.frombuffer(self._out.cpu().numpy().tobytes(), dtype=np.dtype(
            [("n_reveals", "<i8"), ("iterations", "<i4"), ("terminated_by", "<i4"), ("status", "<i4"),
             ("pad", "<i4")]))
        topk = self._topk.cpu().numpy()
        res = []
        NT = self.n_rows * self.n_cols
        for c in range(self.n_local):
            o = out[c]
            if o["status"] == 1:
                raise RuntimeError("internal error: both boundary rows exhausted while unseparated")
            if o["status"] == _lib.CBX_BANDIT_EDESC:
                raise ValueError("descriptor outside the kernel's shape contract")
            if o["status"] != 0:
                raise RuntimeError(f"bandit kernel status {int(o['status'])} (exact-sum capacity exceeded)")
            n = int(o["n_reveals"])
            a = c * NT
            rev = Reveals(self._tr_i[a:a + n].cpu().numpy(), self._tr_t[a:a + n].cpu().numpy(),
                          self._tr_v[a:a + n].cpu().numpy())
            term = "separation" if o["terminated_by"] == _lib.CBX_TERM_SEPARATION else "exhaustion"
            res.append(RunResult([int(x) for x in topk[c]], n / NT, rev, int(o["iterations"]), term))
        return res


def run_local_shards(batch, ranges, cfg: BanditConfig, bounds: CellBounds | tuple[float, float] = (-1.0, 1.0)):
    """Several ranks of a document-sharded run on ONE GPU, as co-resident CTAs of one cooperative launch
    sharing this GPU's copy of the pool: each owns ``ranges[c]`` and exchanges through the others'
    inboxes in device memory — the mailbox protocol of run_mailbox without NVLink (its single-GPU test).
    Returns one RunResult per rank (all identical)."""
    import torch

    run = MailboxRun(batch, ranges, cfg, bounds)
    n = run.n_local
    val = torch.empty((n, run.slots), dtype=torch.float64, device=run.dev)
    flag = torch.zeros((n, run.slots), dtype=torch.int32, device=run.dev)
    inbox = [(val[p].data_ptr(), flag[p].data_ptr()) for p in range(n)]
    run.set_peers([inbox] * n)
    run.launch()
    torch.cuda.current_stream().synchronize()
    res = run.results()
    del val, flag
    return res


def run_mailbox(batch, own: tuple[int, int], cfg: BanditConfig,
                bounds: CellBounds | tuple[float, float] = (-1.0, 1.0), group=None, timing: dict | None = None):
    """This rank's share of a document-sharded run across processes (one GPU each): one persistent launch,
    the per-iteration exchange through NVLink peer memory. Every rank calls it collectively; the inboxes are
    allocated, cleared and mapped (CUDA IPC handles all-gathered over ``group``) before, and released after.
    ``timing``, if given, receives the device time of the launch in ms ("ms")."""
    import torch
    import torch.distributed as dist

    lib = _lib.load()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    run = MailboxRun(batch, [own], cfg, bounds, rank0=rank, n_ranks=world)
    slots = run.slots
    base, nbytes = ctypes.c_void_p(), ctypes.c_size_t()
    _lib.check(lib.cbx_mbox_alloc(slots, ctypes.byref(base), ctypes.byref(nbytes)), "mbox_alloc")
    opened = []
    try:
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(lib.cbx_mbox_clear(base, slots, stream), "mbox_clear")
        h = ctypes.create_string_buffer(_lib.CBX_IPC_HANDLE_BYTES)
        _lib.check(lib.cbx_ipc_get_handle(base, h), "ipc_get_handle")
        handles = [None] * world
        dist.all_gather_object(handles, h.raw, group=group)
        table = []
        for p in range(world):
            if p == rank:
                pb = base
            else:
                pb = ctypes.c_void_p()
                _lib.check(lib.cbx_ipc_open(ctypes.create_string_buffer(handles[p], _lib.CBX_IPC_HANDLE_BYTES),
                                            ctypes.byref(pb)), "ipc_open")
                opened.append(pb)
            v = _lib.CbxMboxPeer()
            _lib.check(lib.cbx_mbox_view(pb, slots, ctypes.byref(v)), "mbox_view")
            table.append((v.val, v.flag))
        run.set_peers([table])
        torch.cuda.current_stream().synchronize()  # this inbox is clear ...
        dist.barrier(group=group)                  # ... and so is every other one: nobody writes early
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run.launch()
        e1.record()
        torch.cuda.current_stream().synchronize()
        if timing is not None:
            timing["ms"] = e0.elapsed_time(e1)
        dist.barrier(group=group)                  # every kernel has finished writing into the inboxes
        return run.results()[0]
    finally:
        for pb in opened:
            lib.cbx_ipc_close(pb)
        lib.cbx_mbox_free(base)
