"""Synthetic workloads with the shapes of BASELINE.json's five configs.

The reference ships no data for these configs (its own generator, synth.py,
draws a different planted-ladder scheme), so this module is the single
definition of the inputs both sides see. Decisions:

* every token is ``unit(x) = x / ||x||_2`` computed in float64, then cast to
  the config dtype; the cast tensor is canonical and the CPU oracle receives
  its exact float64 upcast;
* planted noise is per-coordinate ``sigma / sqrt(d)`` so the noise norm is
  about ``sigma`` (the literal reading buries planted tokens);
* "lognormal mean 180, sigma 0.5" is read as the mean:
  ``mu = ln 180 - 0.5**2 / 2``, rounded and clipped to [16, 512];
* bf16 is produced float64 -> float32 (RNE) -> bf16 (RNE), carried as raw
  uint16 bits so numpy, torch and the device agree on every value.

Two generators implement the same recipe: a numpy one (bit-reproducible on
any host; used for parity fixtures and CPU baselines) and a torch one that
draws whole batches directly in HBM for the benchmark (different random
stream, same distribution; the oracle is then fed device->host copies).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "WorkloadConfig",
    "CONFIGS",
    "QueryCase",
    "gen_query",
    "gen_batch_device",
    "batch_plan",
    "query_blocks",
    "to_float64",
    "bf16_bits_from_f32",
    "bf16_bits_to_f32",
]


@dataclass(frozen=True)
class WorkloadConfig:
    name: str
    n_queries: int
    n_docs: int
    lq: tuple[int, int]          # inclusive range of query lengths
    dim: int
    doc_len: tuple[str, float, float, float]  # ("uniform", lo, hi, _) | ("lognormal", mean, sigma, clip_hi) | ("fixed", L, 0, 0)
    dtype: str                   # "f32" | "f16" | "bf16"
    k: int
    n_relevant: int
    planted_sigma: float
    planted_frac: float
    similarity: str              # oracle construction
    scheme: str = "planted"      # "planted" | "clustered" | "isotropic"
    alphas: tuple[float, ...] = (1.0,)
    seed: int = 0


_LOGN_MU = math.log(180.0) - 0.5 ** 2 / 2.0

CONFIGS: dict[str, WorkloadConfig] = {
    "cfg1": WorkloadConfig("cfg1", 1, 100, (32, 32), 128, ("uniform", 64, 256, 0), "f32", 5,
                           10, 0.8, 0.3, "cosine", seed=0),
    "cfg2": WorkloadConfig("cfg2", 256, 1000, (32, 32), 128, ("lognormal", 180.0, 0.5, 512), "f16", 10,
                           20, 1.0, 0.3, "dot", seed=2),
    "cfg3": WorkloadConfig("cfg3", 128, 500, (16, 48), 128, ("fixed", 1030, 0, 0), "bf16", 5,
                           5, 0.5, 0.3, "dot", scheme="clustered", seed=3),
    "cfg4": WorkloadConfig("cfg4", 1, 100_000, (32, 32), 128, ("lognormal", 180.0, 0.5, 512), "f16", 100,
                           100, 1.0, 0.3, "dot", seed=4),
    "cfg5": WorkloadConfig("cfg5", 64, 2000, (64, 64), 256, ("fixed", 300, 0, 0), "bf16", 20,
                           0, 0.0, 0.0, "dot", scheme="isotropic",
                           alphas=tuple(float(a) for a in np.logspace(-3, 0, 5)), seed=5),
}


def bf16_bits_from_f32(x: np.ndarray) -> np.ndarray:
    """Round float32 to bfloat16 (nearest-even); returns the uint16 bit patterns."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))
    return ((b + rounding) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def _unit(x: np.ndarray) -> np.ndarray:
    return x / np.linalg.norm(x, axis=-1, keepdims=True)


def _cast(x64: np.ndarray, dtype: str) -> np.ndarray:
    """float64 -> canonical storage (float32 / float16 / uint16 bf16 bits)."""
    if dtype == "f32":
        return x64.astype(np.float32)
    if dtype == "f16":
        return x64.astype(np.float16)
    if dtype == "bf16":
        return bf16_bits_from_f32(x64.astype(np.float32))
    raise ValueError(f"unknown dtype {dtype!r}")


def to_float64(stored: np.ndarray, dtype: str) -> np.ndarray:
    """Exact float64 upcast of a canonical-storage array (what the oracle sees)."""
    if dtype == "bf16":
        return bf16_bits_to_f32(stored).astype(np.float64)
    return np.asarray(stored).astype(np.float64)


@dataclass
class QueryCase:
    """One query and its candidate pool in canonical storage, CSR-packed."""

    cfg: WorkloadConfig
    query: np.ndarray            # (Lq, d) canonical storage
    doc_tokens: np.ndarray       # (sum L_i, d) canonical storage
    doc_offsets: np.ndarray      # (N + 1,) int64
    relevant: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))

    @property
    def dtype(self) -> str:
        return self.cfg.dtype

    @property
    def n_docs(self) -> int:
        return len(self.doc_offsets) - 1

    def query64(self) -> np.ndarray:
        return to_float64(self.query, self.dtype)

    def docs64(self) -> list[np.ndarray]:
        flat = to_float64(self.doc_tokens, self.dtype)
        off = self.doc_offsets
        return [flat[off[i]:off[i + 1]] for i in range(self.n_docs)]


def _doc_lengths(cfg: WorkloadConfig, rng: np.random.Generator, n: int) -> np.ndarray:
    kind, a, b, c = cfg.doc_len
    if kind == "uniform":
        return rng.integers(int(a), int(b) + 1, size=n).astype(np.int64)
    if kind == "lognormal":
        mu = math.log(a) - b ** 2 / 2.0
        return np.clip(np.rint(rng.lognormal(mu, b, size=n)), 16, int(c)).astype(np.int64)
    if kind == "fixed":
        return np.full(n, int(a), dtype=np.int64)
    raise ValueError(kind)


def gen_query(cfg: WorkloadConfig | str, q: int = 0, n_docs: int | None = None) -> QueryCase:
    """Deterministically generate query ``q`` of a config (numpy, seed ``(cfg.seed, q)``).

    ``n_docs`` overrides the pool size (smaller parity cases with the same
    recipe); the relevant-doc count is scaled down with it.
    """
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    rng = np.random.default_rng((cfg.seed, q)) if cfg.name != "cfg1" else np.random.default_rng(cfg.seed)
    n = cfg.n_docs if n_docs is None else int(n_docs)
    d = cfg.dim
    lq = int(rng.integers(cfg.lq[0], cfg.lq[1] + 1)) if cfg.lq[0] != cfg.lq[1] else cfg.lq[0]
    query = _unit(rng.standard_normal((lq, d)))
    lengths = _doc_lengths(cfg, rng, n)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lengths, out=offsets[1:])
    total = int(offsets[-1])
    # The tokens are drawn, normalised and cast in row chunks straight into storage: the Generator's normal
    # stream does not depend on how the draw is split and the cast is per element, so the result equals one
    # float64 draw of the whole matrix cast at the end, at a fraction of the memory (cfg4: 4.6 GB of fp16
    # instead of 2 x 18.4 GB of float64).
    if cfg.scheme == "clustered":
        tokens = _unit(rng.standard_normal((total, d)))
    else:
        tokens = np.empty((total, d), dtype=_cast(np.zeros((1, d)), cfg.dtype).dtype)
        chunk = 1 << 18
        for s0 in range(0, total, chunk):
            e = min(total, s0 + chunk)
            tokens[s0:e] = _cast(_unit(rng.standard_normal((e - s0, d))), cfg.dtype)
    n_rel = min(n, int(round(cfg.n_relevant * n / cfg.n_docs))) if cfg.n_relevant else 0
    relevant = np.sort(rng.choice(n, size=n_rel, replace=False)) if n_rel else np.zeros(0, np.int64)
    noise = cfg.planted_sigma / math.sqrt(d)
    if cfg.scheme == "planted":
        for r in relevant:
            L = int(lengths[r])
            m = int(round(cfg.planted_frac * L))
            pos = rng.choice(L, size=m, replace=False)
            ts = rng.integers(0, lq, size=m)
            tokens[offsets[r] + pos] = _cast(_unit(query[ts] + noise * rng.standard_normal((m, d))), cfg.dtype)
        return QueryCase(cfg, _cast(query, cfg.dtype), tokens, offsets, relevant)
    if cfg.scheme == "isotropic":
        return QueryCase(cfg, _cast(query, cfg.dtype), tokens, offsets, relevant)
    elif cfg.scheme == "clustered":
        is_rel = np.zeros(n, dtype=bool)
        is_rel[relevant] = True
        for i in range(n):
            L = int(lengths[i])
            if is_rel[i]:
                ts = rng.integers(0, lq, size=8)
                cent = _unit(query[ts] + noise * rng.standard_normal((8, d)))
            else:
                cent = _unit(rng.standard_normal((8, d)))
            m = int(round(cfg.planted_frac * L))
            pos = rng.choice(L, size=m, replace=False)
            which = rng.integers(0, 8, size=m)
            tokens[offsets[i] + pos] = _unit(cent[which] + noise * rng.standard_normal((m, d)))
    return QueryCase(cfg, _cast(query, cfg.dtype), _cast(tokens, cfg.dtype), offsets, relevant)


def batch_plan(cfg: WorkloadConfig | str, n_queries: int | None = None, seed: int = 0, n_docs: int | None = None):
    """Host side of :func:`gen_batch_device` for the WHOLE batch: per-query lengths (doc lengths [nq, n] and
    query lengths [nq]) from one host generator, so every rank of a sharded run agrees on every query's shape
    and can cut the batch into balanced query blocks before drawing any token."""
    import torch

    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    nq = cfg.n_queries if n_queries is None else int(n_queries)
    n = cfg.n_docs if n_docs is None else int(n_docs)
    gc = torch.Generator()
    gc.manual_seed(int(seed) * 1_000_003 + cfg.seed)
    kind, a, b, c = cfg.doc_len
    if kind == "uniform":
        lens = torch.randint(int(a), int(b) + 1, (nq * n,), generator=gc)
    elif kind == "lognormal":
        mu = math.log(a) - b ** 2 / 2.0
        lens = torch.empty(nq * n, dtype=torch.float64).log_normal_(mu, b, generator=gc).round().clamp_(16, int(c))
        lens = lens.to(torch.int64)
    else:
        lens = torch.full((nq * n,), int(a), dtype=torch.int64)
    lqs = torch.randint(cfg.lq[0], cfg.lq[1] + 1, (nq,), generator=gc)
    return cfg, lens.numpy().reshape(nq, n), lqs.numpy().astype(np.int64)


def query_blocks(lens: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous query blocks [a, b) for `world` ranks, balanced by doc tokens (the scorer's HBM bytes,
    sum L_i * d * s per query)."""
    per_q = np.asarray(lens, dtype=np.int64).reshape(len(lens), -1).sum(axis=1)
    nq = len(per_q)
    off = np.zeros(nq + 1, np.int64)
    np.cumsum(per_q, out=off[1:])
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(off[:nq], (int(off[-1]) * r) // world, side="left")))
    cuts.append(nq)
    cuts = np.maximum.accumulate(np.array(cuts))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def gen_batch_device(cfg: WorkloadConfig | str, n_queries: int | None = None, seed: int = 0, device="cuda",
                     n_docs: int | None = None, queries: tuple[int, int] | None = None):
    """Draw a batch of a config directly in HBM with torch's device RNG.

    Same recipe as :func:`gen_query` (unit Gaussian tokens, planted /
    clustered relevance, lognormal or fixed lengths) but a different random
    stream: parity against the oracle is done on device->host copies.
    Shapes come from :func:`batch_plan`; query q's tokens are drawn from its
    own generator (seeded by (seed, cfg, q)), so ``queries=(a, b)`` yields
    exactly queries a..b-1 of the full batch — what one rank of a
    query-sharded run holds. Returns ``(TokenBatch, host_offsets)`` with host
    copies of the (block-local) offsets.
    """
    import torch

    from .batch import TokenBatch

    cfg, lens_all, lqs_all = batch_plan(cfg, n_queries, seed, n_docs)
    nq_all, n = lens_all.shape
    qa, qb = (0, nq_all) if queries is None else (int(queries[0]), int(queries[1]))
    if not 0 <= qa <= qb <= nq_all:
        raise ValueError(f"query block {queries} outside [0, {nq_all}]")
    nq = qb - qa
    d = cfg.dim
    tdt = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[cfg.dtype]
    lens = lens_all[qa:qb].reshape(-1)
    lqs = lqs_all[qa:qb]
    d_off = np.zeros(nq * n + 1, dtype=np.int64)
    np.cumsum(lens, out=d_off[1:])
    q_off = np.zeros(nq + 1, dtype=np.int64)
    np.cumsum(lqs, out=q_off[1:])
    qd_off = np.arange(0, nq * n + 1, n, dtype=np.int64)
    total = int(d_off[-1])

    def unit_rows(x):
        return x / x.norm(dim=-1, keepdim=True)

    q_tokens = torch.empty(int(q_off[-1]), d, dtype=tdt, device=device)
    d_tokens = torch.empty(total, d, dtype=tdt, device=device)
    noise = cfg.planted_sigma / math.sqrt(d)
    n_rel = min(n, int(round(cfg.n_relevant * n / cfg.n_docs))) if cfg.n_relevant else 0
    step = 1 << 22
    for qi in range(nq):
        q = qa + qi
        qseed = (int(seed) * 1_000_003 + cfg.seed) * 65_537 + q
        g = torch.Generator(device=device)
        g.manual_seed(qseed)
        gc = torch.Generator()
        gc.manual_seed(qseed)
        q_rows = unit_rows(torch.randn(int(lqs[qi]), d, device=device, generator=g))
        q_tokens[int(q_off[qi]):int(q_off[qi + 1])] = q_rows.to(tdt)
        t0, t1 = int(d_off[qi * n]), int(d_off[(qi + 1) * n])
        for s0 in range(t0, t1, step):
            e = min(t1, s0 + step)
            d_tokens[s0:e] = unit_rows(torch.randn(e - s0, d, device=device, generator=g)).to(tdt)
        if not (n_rel and cfg.scheme in ("planted", "clustered")):
            continue
        q_rows = q_tokens[int(q_off[qi]):int(q_off[qi + 1])].float()
        lq = q_rows.shape[0]
        rel = torch.randperm(n, generator=gc)[:n_rel] + qi * n
        for r in rel.tolist():
            s0, L = int(d_off[r]), int(lens[r])
            m = int(round(cfg.planted_frac * L))
            pos = torch.randperm(L, generator=gc)[:m].to(device) + s0
            if cfg.scheme == "planted":
                ts = torch.randint(0, lq, (m,), generator=gc).to(device)
                base = q_rows[ts]
            else:
                ts = torch.randint(0, lq, (8,), generator=gc).to(device)
                cent = unit_rows(q_rows[ts] + noise * torch.randn(8, d, device=device, generator=g))
                base = cent[torch.randint(0, 8, (m,), generator=gc).to(device)]
            d_tokens[pos] = unit_rows(base + noise * torch.randn(m, d, device=device, generator=g)).to(tdt)
    host = (q_off, d_off, qd_off)
    batch = TokenBatch.from_device(q_tokens, torch.from_numpy(q_off).to(device), d_tokens,
                                   torch.from_numpy(d_off).to(device), torch.from_numpy(qd_off).to(device),
                                   clamp_negative=False, host_offsets=host)
    return batch, host
