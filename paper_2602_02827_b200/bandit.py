"""Drop-in Col-Bandit ``run`` executing the whole adaptive loop in one device kernel.

``BanditConfig`` / ``RunResult`` / ``run(oracle, bounds, cfg)`` keep the
reference's fields, defaults, validation, exception types and messages
(colbandit/bandit.py:40-350). The loop itself — warm-up, boundary selection,
epsilon-greedy column choice with numpy's PCG64 stream, float64 reveal,
exact-sum interval update, Top-K maintenance — runs in ``cbx_bandit_run``
(csrc/bandit.cu) without host round trips; the host only seeds the
generator (numpy SeedSequence, as the reference does at bandit.py:193),
evaluates ``log_term`` with ``math.log`` and, for ``static-warmup`` only,
draws the warm-up sample with numpy's ``Generator.choice`` (bandit.py:152).

``run_batch`` launches many independent runs (queries x parameters) at once:
one CTA per run.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .bounds import CellBounds, RadiusConfig

__all__ = ["BanditConfig", "RunResult", "Reveals", "EXPLORE_MODES", "run", "run_batch", "prepare_batch", "launch_batch",
           "ceil_cells", "select_ambiguous",
           "select_token", "static_warmup", "init_one_per_row", "BanditJob"]

EXPLORE_MODES = ("epsilon-greedy", "static-warmup", "uniform-row")
_MODE_CODE = {"epsilon-greedy": _lib.CBX_EPSILON_GREEDY, "static-warmup": _lib.CBX_STATIC_WARMUP,
              "uniform-row": _lib.CBX_UNIFORM_ROW}
MAX_COLS = 128  # CBX_BANDIT_MAX_COLS: two 64-bit unrevealed-column words per row
TREE_ROWS = 0  # pools larger than this select boundary rows through tournament trees (measured faster at every size)


@dataclass(frozen=True)
class BanditConfig:
    """bandit.py:40-76."""

    k: int
    delta: float = 0.01
    alpha_ef: float = 1.0
    epsilon: float = 0.1
    explore_mode: str = "epsilon-greedy"
    gamma_init: float = 0.0
    seed: int | tuple[int, ...] | None = 0
    c: float = 1.0
    union_mode: str = "per-document"

    def __post_init__(self) -> None:
        if self.k < 0:
            raise ValueError(f"k must be non-negative, got {self.k}")
        if not 0.0 <= self.epsilon <= 1.0:
            raise ValueError(f"epsilon must be in [0, 1], got {self.epsilon}")
        if self.explore_mode not in EXPLORE_MODES:
            raise ValueError(f"explore_mode must be one of {EXPLORE_MODES}, got {self.explore_mode!r}")
        if not 0.0 <= self.gamma_init <= 1.0:
            raise ValueError(f"gamma_init must be in [0, 1], got {self.gamma_init}")
        self.radius_config

    @property
    def radius_config(self) -> RadiusConfig:
        return RadiusConfig(self.alpha_ef, self.delta, self.c, self.union_mode)


class Reveals(Sequence):
    """The reveal trace of a run as three numpy columns (row i int32, column t int32, value float64).

    Behaves like the reference's ``list[tuple[int, int, float]]`` (bandit.py:79-95): indexing yields
    ``(int, int, float)`` tuples, slicing yields a list, and it compares equal to a list of tuples with the
    same entries; the Python tuples are only built when they are asked for, so fetching a large batch of
    runs costs one compact device-to-host copy instead of a tuple per revealed cell.
    """

    __slots__ = ("i", "t", "v", "_list")

    def __init__(self, i, t, v):
        self.i = np.asarray(i, dtype=np.int32)
        self.t = np.asarray(t, dtype=np.int32)
        self.v = np.asarray(v, dtype=np.float64)
        self._list = None

    @classmethod
    def from_list(cls, reveals) -> "Reveals":
        if isinstance(reveals, Reveals):
            return reveals
        n = len(reveals)
        a = np.array([(i, t) for i, t, _ in reveals], dtype=np.int32).reshape(n, 2)
        return cls(a[:, 0], a[:, 1], np.array([v for *_, v in reveals], dtype=np.float64))

    def tolist(self) -> list:
        if self._list is None:
            self._list = list(zip(self.i.tolist(), self.t.tolist(), self.v.tolist()))
        return self._list

    def __len__(self) -> int:
        return len(self.i)

    def __getitem__(self, k):
        if isinstance(k, slice):
            return self.tolist()[k]
        return (int(self.i[k]), int(self.t[k]), float(self.v[k]))

    def __iter__(self):
        return iter(self.tolist())

    def __eq__(self, other):
        if isinstance(other, Reveals):
            return (len(self) == len(other) and np.array_equal(self.i, other.i) and np.array_equal(self.t, other.t)
                    and np.array_equal(self.v, other.v))
        if isinstance(other, (list, tuple)):
            return len(other) == len(self) and self.tolist() == [tuple(x) for x in other]
        return NotImplemented

    def __ne__(self, other):
        eq = self.__eq__(other)
        return eq if eq is NotImplemented else not eq

    __hash__ = None

    def __repr__(self) -> str:
        return repr(self.tolist()) if len(self) <= 8 else f"Reveals({len(self)} cells: {self[:3]!r} ...)"


@dataclass(frozen=True)
class RunResult:
    """bandit.py:79-95 (``reveals`` is a :class:`Reveals`, which compares equal to the reference's list)."""

    topk: list[int]
    coverage: float
    reveals: Sequence[tuple[int, int, float]]
    iterations: int
    terminated_by: str


def ceil_cells(fraction: float, total: int) -> int:
    """bandit.py:98-108 (snaps near-integer products before the ceiling)."""
    x = fraction * total
    nearest = round(x)
    if abs(x - nearest) < 1e-9 * max(1.0, total):
        return int(nearest)
    return math.ceil(x)


def select_ambiguous(i_plus: int, i_minus: int, width_plus: float, width_minus: float) -> int:
    return i_plus if width_plus >= width_minus else i_minus


def select_token(ledger, bounds: CellBounds, i: int, epsilon: float, rng: np.random.Generator) -> int:
    """bandit.py:116-136 — an unrevealed column of row i: uniform with probability epsilon (the draw is
    always made), else the widest support, ties to the lowest column. Host helper for ledger-driven callers;
    the device loop makes the same choice in cbx_bandit_run."""
    cols = ledger.unobserved_cols(i)
    if not cols:
        raise ValueError(f"row {i} is fully revealed; no column to select")
    if rng.random() < epsilon:
        return cols[int(rng.integers(len(cols)))]
    widths = bounds.hi[i, cols] - bounds.lo[i, cols]
    return cols[int(np.argmax(widths))]


def static_warmup(oracle, ledger, gamma_init: float, rng: np.random.Generator):
    """bandit.py:139-156 — reveal ceil(gamma_init * N * T) cells uniformly without replacement."""
    from .oracle import reveal

    if not 0.0 <= gamma_init <= 1.0:
        raise ValueError(f"gamma_init must be in [0, 1], got {gamma_init}")
    total = ledger.n_rows * ledger.n_cols
    m = ceil_cells(gamma_init, total)
    if m == 0:
        return ledger
    for f in rng.choice(total, size=m, replace=False):
        i, t = divmod(int(f), ledger.n_cols)
        reveal(ledger, oracle, i, t)
    return ledger


def init_one_per_row(oracle, ledger, rng: np.random.Generator):
    """bandit.py:159-166 — one uniformly random cell per row (the epsilon-greedy warm start)."""
    from .oracle import reveal

    for i in range(ledger.n_rows):
        reveal(ledger, oracle, i, int(rng.integers(ledger.n_cols)))
    return ledger


@dataclass
class BanditJob:
    """One run of a batched launch: a query (or matrix block) + bounds + config."""

    cfg: BanditConfig
    n_rows: int
    n_cols: int
    query: int = 0          # token source: query index in the batch
    row_begin: int = 0      # global doc index (token source) / matrix row of row 0
    bounds: CellBounds | tuple[float, float] = (-1.0, 1.0)
    selection: str = "auto"  # "scan" | "tree" | "auto" (= tree for pools above TREE_ROWS)


_PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
_M128 = (1 << 128) - 1
_M64 = (1 << 64) - 1
_SEED_CACHE: dict = {}


def pcg64_seed_state(seed) -> tuple[int, int]:
    """(state, inc) of ``np.random.Generator(PCG64(seed))`` right after seeding, without building a Generator.

    numpy's PCG64 takes four 64-bit words from ``SeedSequence(seed).generate_state(4, uint64)``: initstate =
    w0:w1, initseq = w2:w3, then pcg_setseq_128_srandom_r — state = 0, inc = initseq << 1 | 1, step, state +=
    initstate, step (step: state = state * MULT + inc mod 2^128). ~4x cheaper than default_rng(seed), and
    cached per seed (a sweep reuses each query's seed for every alpha). Checked against numpy in the tests.
    """
    key = seed if not isinstance(seed, list) else tuple(seed)
    try:
        return _SEED_CACHE[key]
    except (KeyError, TypeError):
        pass
    w = [int(x) for x in np.random.SeedSequence(seed).generate_state(4, np.uint64)]
    initstate, initseq = (w[0] << 64) | w[1], (w[2] << 64) | w[3]
    inc = ((initseq << 1) | 1) & _M128
    state = inc  # 0 * MULT + inc
    state = (state + initstate) & _M128
    state = (state * _PCG_MULT + inc) & _M128
    try:
        if len(_SEED_CACHE) > 65536:
            _SEED_CACHE.clear()
        _SEED_CACHE[key] = (state, inc)
    except TypeError:
        pass
    return state, inc


def _rng_state(seed, explore_mode, gamma_init, total_cells):
    """numpy seeding (+ the static warm-up draw) on the host; returns (pcg64 struct, warm cells)."""
    warm = np.zeros(0, dtype=np.int32)
    p = _lib.CbxPcg64()
    m = ceil_cells(gamma_init, total_cells) if explore_mode == "static-warmup" else 0
    if m == 0 and seed is not None:
        s, inc = pcg64_seed_state(seed)
        has32, buf = 0, 0
    else:
        g = np.random.default_rng(seed)
        if m:
            warm = np.asarray(g.choice(total_cells, size=m, replace=False), dtype=np.int32)
        st = g.bit_generator.state
        s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
        has32, buf = int(st["has_uint32"]), int(st["uinteger"])
    p.state_hi, p.state_lo = s >> 64, s & _M64
    p.inc_hi, p.inc_lo = inc >> 64, inc & _M64
    p.has_uint32 = has32
    p.uinteger = buf
    return p, warm


def _sm_count() -> int:
    import torch

    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def _warms_up(job: BanditJob, uniform) -> bool:
    """Will the run reach its lazy warm-up (i.e. fail the stop test at iteration 1, bandit.py:281-296)?

    Only decides whether the warm-up cells are computed ahead by cbx_bandit_prewarm (a performance
    choice): a run that is not pre-warmed computes them inside the loop kernel, so a borderline case is
    answered False. Initial intervals: LCB = sum(lo), UCB = sum(hi), proxy = midpoint (bounds.py:211-263).
    """
    cfg, N = job.cfg, job.n_rows
    if cfg.explore_mode == "uniform-row" or cfg.k >= N:
        return False
    if uniform:
        return uniform[0] < uniform[1]
    b = job.bounds
    h_lo, h_hi = b.lo.sum(axis=1), b.hi.sum(axis=1)
    proxy = 0.5 * (h_lo + h_hi)
    order = np.lexsort((np.arange(N), -proxy))
    top, rest = order[: cfg.k], order[cfg.k:]
    lcb_plus, ucb_minus = h_lo[top].min(), h_hi[rest].max()
    return bool(lcb_plus < ucb_minus - 1e-9 * (abs(lcb_plus) + abs(ucb_minus) + 1.0))


def _desc_dtype() -> np.dtype:
    """numpy view of cbx_bandit_run_desc (field offsets taken from the ctypes mirror of the header)."""
    names, formats, offsets = [], [], []
    for name, ct in _lib.CbxBanditRunDesc._fields_:
        off = getattr(_lib.CbxBanditRunDesc, name).offset
        if name == "rng":
            for sub, sct in _lib.CbxPcg64._fields_:
                names.append("rng_" + sub)
                formats.append(np.dtype(sct))
                offsets.append(off + getattr(_lib.CbxPcg64, sub).offset)
            continue
        names.append(name)
        formats.append(np.dtype(ct))
        offsets.append(off)
    return np.dtype({"names": names, "formats": formats, "offsets": offsets,
                     "itemsize": ctypes.sizeof(_lib.CbxBanditRunDesc)})


_DESC_DTYPE = None
_LOG_TERM_CACHE: dict = {}


def _log_term(cfg: BanditConfig, N: int, T: int) -> float:
    key = (cfg.delta, cfg.c, cfg.union_mode, cfg.alpha_ef, N, T)
    v = _LOG_TERM_CACHE.get(key)
    if v is None:
        if len(_LOG_TERM_CACHE) > 65536:
            _LOG_TERM_CACHE.clear()
        v = _LOG_TERM_CACHE[key] = cfg.radius_config.log_term(N, T)
    return v


def prepare_batch(jobs: Sequence[BanditJob], batch=None, matrix=None, prewarm: bool | None = None,
                  row_cache: bool | int = False) -> dict:
    """Host side of a batched launch: validate the jobs, seed the generators, build the run descriptors and
    move them (and any per-cell bounds) to the device; outputs are allocated. ``launch_batch`` then issues
    the kernels. ``prewarm`` (None = auto: when the runs fit one CTA per SM) computes the warm-up cells of
    token-backed runs with one HBM-bound cbx_bandit_prewarm launch ahead of the loop kernel (same values,
    same traces). The descriptors are filled column-wise into a numpy view of cbx_bandit_run_desc (one
    host->device copy), so preparing a few hundred runs costs well under the kernel's time."""
    global _DESC_DTYPE
    torch = _lib.require_cuda()
    lib = _lib.load()
    if batch is None and matrix is None:
        raise ValueError("need a TokenBatch or a device matrix as the cell source")
    if _DESC_DTYPE is None:
        _DESC_DTYPE = _desc_dtype()
    n = len(jobs)
    cols = {k: [] for k in ("query", "row_begin", "n_rows", "n_cols", "k", "explore_mode", "n_warm", "flags",
                            "warm_off", "alpha_ef", "epsilon", "log_term", "bounds_off", "lo_uniform", "hi_uniform",
                            "trace_off", "state_off")}
    rngs = []
    lo_parts, hi_parts, warm_parts = [], [], []
    b_off = w_off = tr_off = st_off = 0
    max_rows = max_k = 1
    results: list = [None] * n
    live = []
    warm_counts = []
    # the in-loop warm-up gathers with one CTA; with at most one run per SM that CTA is latency bound and
    # a grid-wide pre-pass wins (measured: cfg3 128 runs, cfg4 1 run); with more runs the loop kernels
    # already keep HBM busy during their warm-ups (cfg2 256 runs: no gain)
    prewarm_on = prewarm if prewarm is not None else len(jobs) <= _sm_count()
    for r, job in enumerate(jobs):
        cfg = job.cfg
        N, T = int(job.n_rows), int(job.n_cols)
        if T > MAX_COLS:
            raise ValueError(f"the device bandit supports at most {MAX_COLS} query tokens, got {T}")
        if cfg.k > N:
            raise ValueError(f"k={cfg.k} exceeds the number of documents ({N})")
        if cfg.k == 0:
            results[r] = RunResult([], 0.0, [], 0, "separation")
            continue
        if job.selection not in ("auto", "scan", "tree"):
            raise ValueError(f"selection must be 'auto', 'scan' or 'tree', got {job.selection!r}")
        live.append(r)
        cols["query"].append(job.query)
        cols["row_begin"].append(job.row_begin)
        cols["n_rows"].append(N)
        cols["n_cols"].append(T)
        cols["k"].append(cfg.k)
        cols["explore_mode"].append(_MODE_CODE[cfg.explore_mode])
        cols["alpha_ef"].append(cfg.alpha_ef)
        cols["epsilon"].append(cfg.epsilon)
        cols["log_term"].append(_log_term(cfg, N, T))
        bnd = job.bounds
        uni = bnd if isinstance(bnd, tuple) else bnd.uniform_values()
        if uni:
            cols["bounds_off"].append(-1)
            cols["lo_uniform"].append(uni[0])
            cols["hi_uniform"].append(uni[1])
        else:
            cols["bounds_off"].append(b_off)
            cols["lo_uniform"].append(0.0)
            cols["hi_uniform"].append(0.0)
            lo_parts.append(np.ascontiguousarray(bnd.lo, dtype=np.float64).ravel())
            hi_parts.append(np.ascontiguousarray(bnd.hi, dtype=np.float64).ravel())
            b_off += N * T
        p, warm = _rng_state(cfg.seed, cfg.explore_mode, cfg.gamma_init, N * T)
        rngs.append((p.state_hi, p.state_lo, p.inc_hi, p.inc_lo, p.has_uint32, p.uinteger))
        cols["n_warm"].append(len(warm))
        cols["warm_off"].append(w_off)
        warm_parts.append(warm)
        w_off += len(warm)
        tree = job.selection == "tree" or (job.selection == "auto" and N > TREE_ROWS)
        flags = _lib.CBX_BANDIT_TREE if tree else 0
        pre = prewarm_on and batch is not None and _warms_up(job, uni)
        if pre:
            flags |= _lib.CBX_BANDIT_PREWARMED
        cols["flags"].append(flags)
        warm_counts.append((N if cfg.explore_mode == "epsilon-greedy" else len(warm)) if pre else 0)
        cols["trace_off"].append(tr_off)
        cols["state_off"].append(st_off)
        tr_off += N * T
        st_off += N + _lib.CBX_BANDIT_ROW_SLACK
        max_rows, max_k = max(max_rows, N), max(max_k, cfg.k)
    nl = len(live)
    if nl == 0:
        return dict(results=results, live=live)
    descs = np.zeros(nl, dtype=_DESC_DTYPE)
    for k, v in cols.items():
        descs[k] = v
    rng_a = np.array(rngs, dtype=np.uint64)
    for j, sub in enumerate(("state_hi", "state_lo", "inc_hi", "inc_lo", "has_uint32", "uinteger")):
        descs["rng_" + sub] = rng_a[:, j]
    dev = torch.device("cuda", torch.cuda.current_device())
    desc_t = torch.from_numpy(descs.view(np.uint8).reshape(-1)).to(dev)
    lo_t = torch.from_numpy(np.concatenate(lo_parts)).to(dev) if lo_parts else None
    hi_t = torch.from_numpy(np.concatenate(hi_parts)).to(dev) if hi_parts else None
    warm_t = torch.from_numpy(np.concatenate(warm_parts)).to(dev) if w_off else None
    state_bytes = lib.cbx_bandit_state_bytes(st_off)
    state = torch.empty(state_bytes, dtype=torch.uint8, device=dev)
    topk_t = torch.empty((nl, max_k), dtype=torch.int32, device=dev)
    tr_i = torch.empty(max(tr_off, 1), dtype=torch.int32, device=dev)
    tr_t = torch.empty(max(tr_off, 1), dtype=torch.int32, device=dev)
    tr_v = torch.empty(max(tr_off, 1), dtype=torch.float64, device=dev)
    out_t = torch.empty(nl * ctypes.sizeof(_lib.CbxBanditOut), dtype=torch.uint8, device=dev)
    # row-cache variant (reported separately from the on-demand loop): float64 cells of the rows touched by
    # adaptive reveals, same offsets as the trace buffers, plus a filled flag per state row
    rc = None
    if row_cache is not False and row_cache is not None and batch is not None:
        # True: fill a row on the reveal that finds 2 of its cells already revealed; an int sets that count
        thr = 2 if row_cache is True else int(row_cache)
        rc = (torch.empty(max(tr_off, 1), dtype=torch.float64, device=dev),
              torch.zeros(max(st_off, 1), dtype=torch.uint8, device=dev), thr)
    if batch is not None:
        batch.norm_max()  # the fp32 reveal screen's error bound (cbx_batch.d_norm_max), computed once per batch
    bstruct = batch.struct() if batch is not None else None
    ld = matrix.shape[1] if matrix is not None else 0
    wprefix = None
    if sum(warm_counts):
        wp = np.zeros(nl + 1, np.int64)
        np.cumsum(warm_counts, out=wp[1:])
        wprefix = torch.from_numpy(wp).to(dev)
    return dict(results=results, live=live, descs=descs, nl=nl, max_rows=max_rows, max_k=max_k, bstruct=bstruct,
                batch=batch, matrix=matrix, ld=ld, desc_t=desc_t, lo_t=lo_t, hi_t=hi_t, warm_t=warm_t, state=state,
                state_bytes=state_bytes, topk=topk_t, tr_i=tr_i, tr_t=tr_t, tr_v=tr_v, out=out_t, wprefix=wprefix,
                n_prewarm=int(sum(warm_counts)), row_cache=rc)


def launch_batch(p: dict):
    """Issue a prepared batch on the current stream (no host synchronisation); returns the raw outputs."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    bref = ctypes.byref(p["bstruct"]) if p["bstruct"] is not None else None
    if p["wprefix"] is not None:
        _lib.check(lib.cbx_bandit_prewarm(
            bref, p["desc_t"].data_ptr(), p["nl"], p["wprefix"].data_ptr(), p["n_prewarm"], ptr(p["warm_t"]),
            p["tr_i"].data_ptr(), p["tr_t"].data_ptr(), p["tr_v"].data_ptr(), stream), "bandit_prewarm")
    m = p["matrix"]
    rc = p.get("row_cache")
    if rc is not None:
        rc[1].zero_()
        lib.cbx_bandit_set_row_cache(rc[0].data_ptr(), rc[1].data_ptr())
        lib.cbx_bandit_set_row_cache_threshold(rc[2])
    try:
        _launch_run(lib, p, m, bref, ptr, stream)
    finally:
        if rc is not None:
            lib.cbx_bandit_set_row_cache(None, None)
    return dict(descs=p["descs"], live=p["live"], topk=p["topk"], tr_i=p["tr_i"], tr_t=p["tr_t"], tr_v=p["tr_v"],
                out=p["out"], keep=p)


def _launch_run(lib, p, m, bref, ptr, stream):
    _lib.check(lib.cbx_bandit_run(
        bref, m.data_ptr() if m is not None else None, p["ld"], p["desc_t"].data_ptr(), p["nl"], p["max_rows"],
        ptr(p["lo_t"]), ptr(p["hi_t"]), ptr(p["warm_t"]), p["state"].data_ptr(), p["state_bytes"],
        p["topk"].data_ptr(), p["max_k"], p["tr_i"].data_ptr(), p["tr_t"].data_ptr(), p["tr_v"].data_ptr(),
        p["out"].data_ptr(), stream), "bandit_run")


def run_batch(jobs: Sequence[BanditJob], batch=None, matrix=None, return_traces: bool = True, sync: bool = True,
              prewarm: bool | None = None, row_cache: bool | int = False, stats: dict | None = None):
    """Launch every job in one kernel; returns a list of RunResult (or raw device outputs if sync=False).

    ``row_cache=True`` selects the row-cache variant for token-backed runs with generic bounds: a reveal that
    finds two cells of its row already revealed (an int sets another count; 0 = first touch) computes ALL of
    the row's cells from one gather of the document — the reference's oracle does that on first touch,
    oracle.py:205-215 — and later reveals of the row read them back. Results and
    traces are identical to the on-demand loop; it gathers fewer bytes and does more arithmetic per gather,
    so it is accounted separately (``stats["rows_filled"]``: gathers of whole rows, per run)."""
    p = prepare_batch(jobs, batch, matrix, prewarm, row_cache)
    if not p["live"]:
        return p["results"]
    raw = launch_batch(p)
    if not sync:
        return raw
    return collect(raw, jobs, p["results"], return_traces, stats)


_STAGE = {}


def _pinned_stage(nbytes: int):
    """A grow-only pinned host buffer for trace copies (allocating pinned memory per call costs milliseconds)."""
    import torch

    t = _STAGE.get("buf")
    if t is None or t.numel() < nbytes:
        t = _STAGE["buf"] = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
    return t


def collect(raw, jobs, results=None, return_traces: bool = True, stats: dict | None = None):
    """Fetch a launch's device outputs and build RunResults (raises on device-side errors)."""
    if results is None:
        results = [None] * len(jobs)
    import torch

    live = raw["live"]
    out = np.frombuffer(raw["out"].cpu().numpy().tobytes(), dtype=np.dtype(
        [("n_reveals", "<i8"), ("iterations", "<i4"), ("terminated_by", "<i4"), ("status", "<i4"), ("pad", "<i4")]))
    if stats is not None:
        stats["rows_filled"] = out["pad"].astype(np.int64)  # row-cache variant: whole-row gathers per live run
        stats["live"] = list(live)
    topk = raw["topk"].cpu().numpy()
    if return_traces:
        # only the used prefix of every run's N*T trace slots crosses PCIe: gather them on the device first
        nrev = out["n_reveals"].astype(np.int64)
        starts = np.asarray(raw["descs"]["trace_off"], dtype=np.int64)
        cum = np.zeros(len(live) + 1, np.int64)
        np.cumsum(nrev, out=cum[1:])
        dev = raw["tr_i"].device
        total = int(cum[-1])
        if total:
            # one device gather of the used slots, two D2H copies into pinned memory, one synchronisation
            # slot -> trace position: per-run shifts expanded on the device (a few hundred values cross PCIe)
            small = torch.from_numpy(np.stack([starts - cum[:-1], nrev])).to(dev)
            pos = torch.arange(total, dtype=torch.int64, device=dev) + \
                torch.repeat_interleave(small[0], small[1], output_size=total)
            blk = torch.empty((total, 4), dtype=torch.int32, device=dev)  # (i, t, v lo word, v hi word)
            blk[:, 0] = raw["tr_i"][pos]
            blk[:, 1] = raw["tr_t"][pos]
            blk[:, 2:].view(torch.float64)[:, 0] = raw["tr_v"][pos]
            stage = _pinned_stage(total * 16)[: total * 16].view(torch.int32).view(total, 4)
            stage.copy_(blk, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            h = stage.numpy().copy()  # the results own their memory; the pinned stage is reused
            tr_i, tr_t, tr_v = h[:, 0], h[:, 1], h[:, 2:].view(np.float64)[:, 0]
        else:
            tr_i, tr_t, tr_v = np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.float64)
    for slot, r in enumerate(live):
        job, o = jobs[r], out[slot]
        if o["status"] == 1:
            raise RuntimeError("internal error: both boundary rows exhausted while unseparated")
        if o["status"] == _lib.CBX_BANDIT_EDESC:
            raise ValueError(f"run {r}: descriptor outside the kernel's shape contract (n_rows >= 1, "
                             f"1 <= n_cols <= {MAX_COLS}, 1 <= k <= n_rows)")
        if o["status"] != 0:
            raise RuntimeError(f"bandit kernel status {int(o['status'])} (exact-sum capacity exceeded)")
        nrev = int(o["n_reveals"])
        reveals = []
        if return_traces:
            a, b = int(cum[slot]), int(cum[slot + 1])
            reveals = Reveals(tr_i[a:b], tr_t[a:b], tr_v[a:b])
        term = "separation" if o["terminated_by"] == _lib.CBX_TERM_SEPARATION else "exhaustion"
        results[r] = RunResult([int(x) for x in topk[slot, : job.cfg.k]], nrev / (job.n_rows * job.n_cols),
                               reveals, int(o["iterations"]), term)
    return results


def run(oracle, bounds: CellBounds, cfg: BanditConfig) -> RunResult:
    """Identify the Top-K rows revealing as few cells as the intervals allow (bandit.py:169-350)."""
    n_rows, n_cols = oracle.n_docs, oracle.n_query_tokens
    if (bounds.n_rows, bounds.n_cols) != (n_rows, n_cols):
        raise ValueError(
            f"bounds shape ({bounds.n_rows}, {bounds.n_cols}) does not match matrix shape ({n_rows}, {n_cols})")
    if cfg.k > n_rows:
        raise ValueError(f"k={cfg.k} exceeds the number of documents ({n_rows})")
    if cfg.k == 0:
        return RunResult([], 0.0, [], 0, "separation")
    if not hasattr(oracle, "_batch"):
        raise TypeError("run() needs a paper_2602_02827_b200 MaxSimOracle (device-resident cells)")
    job = BanditJob(cfg, n_rows, n_cols, 0, 0, bounds)
    if oracle._batch is not None:
        res = run_batch([job], batch=oracle._batch)[0]
    else:
        res = run_batch([job], matrix=oracle._dev_matrix)[0]
    oracle._reveal_count += len(res.reveals)
    return res
