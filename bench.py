#!/usr/bin/env python
"""Benchmark of the B200 MaxSim reranker — the driver's contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

One "step" = one pass of the hot path over one batch: the MaxSim score of
every candidate of every query (tcgen05 dense scorer, P1) + per-query Top-K.
The workload is BASELINE.json configs[1] ("cfg2": 256 queries x 1000
candidates, Lq = 32, d = 128, fp16, lognormal doc lengths, K = 10), drawn on
the device (synthetic; every query from its own seeded generator). Inputs
(11.7 GB of doc tokens) exceed L2 (126 MB), so no flush is needed between
steps.

Multi-GPU (one process per GPU): under torchrun the ranks come from the
environment; ``--gpus N`` without WORLD_SIZE spawns the N ranks itself
(127.0.0.1 rendezvous, NCCL). The 256 queries are STRONG-scaled: rank r holds
the contiguous query block workloads.query_blocks(...)[r], balanced by doc
tokens, and no collective touches the data path (the queries are
independent); value = all queries' cells / max-over-ranks time.

The JSON line also carries the Col-Bandit loop (P2) on the same batch
("bandit": one CTA per query, default BanditConfig, seed (0, q)), with its
revealed-cell throughput, gather bandwidth and CPU-oracle parity; cfg4's
document-sharded exhaustive Top-K ("p1_sharded": per-rank scorer + local
Top-100, one NCCL all-gather of 100 (score, id) pairs per rank, device merge);
the Stage-1 scan + reranker facade ("stage1"); and cfg4's document-sharded
Col-Bandit ("bandit_sharded").

``--impl reference`` times the reference's CPU algorithm (the oracle port in
oracle/maxsim_ref: float64 GEMM + column max + math.fsum + lexsort) on the
box's host cores, one process per core, for the same metric and config.
``--dry-run`` exercises the launcher, the query sharding and the max-over-ranks
reduction without a GPU (gloo; the CPU test of the multi-rank path).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MaxSim cells/sec (exhaustive rerank, oracle-matching Top-K)"
UNIT = "cells/s"
_T0 = time.perf_counter()


def _log(msg: str) -> None:
    """Progress to stderr (stdout carries the one JSON line): where the time goes, and where a stuck run stopped."""
    if int(os.environ.get("RANK", "0")) == 0:
        print(f"bench [{time.perf_counter() - _T0:7.1f} s] {msg}", file=sys.stderr, flush=True)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """SM clock + clock-event reasons sampled through NVML every 5 ms during the timed region."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self.error = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            self.nv = None
            self.error = str(e)

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.samples.append((sm, reasons))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception as e:  # pragma: no cover
                self.error = str(e)
                return
            self._stop.wait(0.005)

    def __enter__(self):
        if self.nv is not None:
            self._sample()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=5)
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {self.error}"]}
        import statistics

        nv = self.nv
        active = set()
        for _, r in self.samples:
            for name, attr in self.REASONS.items():
                if r & getattr(nv, attr):
                    active.add(name)
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_sm,
                "reasons": sorted(active), "samples": len(self.samples)}


# ---------------------------------------------------------------------------- helpers
def _query_host(batch, host_off, q):
    """float64 copies of query q and its documents (for the CPU oracle)."""
    qo, do, qd = host_off
    d0, d1 = int(qd[q]), int(qd[q + 1])
    qt = batch.q_tokens[int(qo[q]):int(qo[q + 1])].double().cpu().numpy()
    dt = batch.d_tokens[int(do[d0]):int(do[d1])].double().cpu().numpy()
    docs = [dt[int(do[i] - do[d0]):int(do[i + 1] - do[d0])] for i in range(d0, d1)]
    return qt, docs


def _blas_one_thread():
    try:
        from threadpoolctl import threadpool_limits

        return threadpool_limits(1)
    except Exception:  # pragma: no cover
        return None


# ---------------------------------------------------------------------------- collectives
def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


def _reduce(values, op="max"):
    """All-reduce a list of floats over the ranks (float64; NCCL or gloo); identity at world 1."""
    import torch

    dist = _dist()
    if dist is None:
        return [float(v) for v in values]
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return t.cpu().tolist()


def _barrier():
    dist = _dist()
    if dist is not None:
        dist.barrier()


# ---------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2602_02827_b200 import workloads as W
    from paper_2602_02827_b200.batch import HostBatch, maxsim_scores, rerank_topk_host, topk

    torch.cuda.set_device(local_rank)
    cfg, lens_all, lqs_all = W.batch_plan(args.config, args.queries, seed=0)
    nq_all = len(lqs_all)
    if nq_all < world:
        raise ValueError(f"{nq_all} queries cannot be sharded over {world} ranks")
    blocks = W.query_blocks(lens_all, world)
    qa, qb = blocks[rank]
    batch, host_off = W.gen_batch_device(cfg, n_queries=args.queries, seed=0, queries=(qa, qb))
    torch.cuda.synchronize()
    nq, K = batch.n_queries, cfg.k
    elem = batch.d_tokens.element_size()
    qo, do, qd = host_off
    lq = np.diff(qo)
    ndocs = np.diff(qd)
    qtok = do[qd[1:]] - do[qd[:-1]]
    cells_total = int(lens_all.shape[1] * lqs_all.sum())  # every query of the job, all ranks
    alg_bytes = int(batch.d_tokens.numel() * elem + batch.q_tokens.numel() * elem + 4 * batch.n_docs)
    alg_flops = int(2 * (qtok * lq).sum() * batch.dim)
    hbm_peak, tf_peak, peak_kind = _peaks()
    stream = torch.cuda.current_stream()
    scores = torch.empty(batch.n_docs, dtype=torch.float32, device="cuda")

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        maxsim_scores(batch, out=scores)
        if ev is not None:
            ev[1].record(stream)
        res = topk(scores, batch.q_doc_off, K, batch.max_q_docs)
        if ev is not None:
            ev[2].record(stream)
        return res

    _log(f"batch of {nq} queries on rank {rank} generated; P1 timed region")
    # ------------------------------------------------ P1, device-resident inputs
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    _barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        start.record(stream)
        for i in range(args.steps):
            idx, val = step(evs[i])
        stop.record(stream)
        torch.cuda.synchronize()
    _barrier()
    ms_step = _reduce([start.elapsed_time(stop)])[0] / args.steps
    kern_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    topk_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps

    result = None
    if rank == 0:
        achieved = alg_bytes / (kern_ms / 1e3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath) and world == 1:
            traffic = json.load(open(tpath)).get(args.config)
        result = {
            "metric": METRIC, "value": cells_total / (ms_step / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype,
            "data": "synthetic (device RNG per query, BASELINE.json configs[1] recipe)",
            "config": {"workload": f"{cfg.name}: {nq_all} queries x {cfg.n_docs} docs, Lq={cfg.lq[0]}, d={cfg.dim}, "
                                   f"lognormal lengths (mean 180, sigma 0.5, clip [16,512]), {cfg.dtype}, K={K}",
                       "queries": nq_all, "query_blocks": blocks,
                       "doc_tokens": int(lens_all.sum()), "doc_tokens_rank0": int(batch.d_tokens.shape[0]),
                       "l2": "inputs (%.1f GB per rank) exceed L2 (126 MB); no flush" % (alg_bytes / 1e9),
                       "parallelism": f"query-sharded x{world}, blocks balanced by doc tokens (no collective)"},
            "queries_per_s": nq_all / (ms_step / 1e3),
            "scorer_ms": kern_ms, "topk_ms": topk_ms,
            "roofline": {"bound": "hbm", "kernel": "maxsim_tc_kernel (rank 0)", "achieved": achieved,
                         "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak, "peak_kind": peak_kind,
                         "alg_bytes_per_launch": alg_bytes, "traffic": traffic,
                         "tensor_tflops": alg_flops / (kern_ms / 1e3) / 1e12, "tensor_peak": tf_peak},
            "clocks": clocks.summary(),
            "gpu_launches": args.steps * 2,
        }

    _log("P1 parity + 1-core CPU baseline")
    # ------------------------------------------------ P1 parity on sampled queries + CPU baseline
    if rank == 0:
        from oracle import maxsim_ref

        lim = _blas_one_thread()
        idx_h, sc_h = idx.cpu().numpy(), scores.cpu().numpy()
        ok, n_chk, cpu_cells, cpu_s = True, 0, 0, 0.0
        for q in range(nq):
            qt, docs = _query_host(batch, host_off, q)
            t0 = time.perf_counter()
            ref_s, ref_t, _ = maxsim_ref.score_query(qt, docs, K)
            cpu_s += time.perf_counter() - t0
            cpu_cells += len(docs) * qt.shape[0]
            d0 = int(qd[q])
            ok &= bool(np.allclose(sc_h[d0:d0 + len(docs)], ref_s, rtol=1e-3, atol=0))
            for g_, r_ in zip(idx_h[q].tolist(), ref_t):
                if g_ != r_ and abs(ref_s[g_] - ref_s[r_]) > 1e-3 * abs(ref_s[r_]):
                    ok = False
            n_chk += 1
            if n_chk >= args.check_queries and cpu_s >= args.cpu_seconds:
                break
        result["parity"] = {"queries_checked": n_chk, "scores_rtol": 1e-3, "topk_match": ok}
        if world == 1 and not args.no_cpu:
            result["cpu_baseline"] = {"value": cpu_cells / cpu_s, "unit": UNIT, "cores": 1, "kind": "port",
                                      "sample": f"{n_chk} {cfg.name} queries through oracle/maxsim_ref (float64 GEMM "
                                                f"+ column max + math.fsum + lexsort, BLAS 1 thread), {cpu_s:.1f} s"}
        del lim
    _barrier()

    # ------------------------------------------------ end-to-end through the public host API
    # The reranking service keeps the corpus resident in HBM (Corpus = ColBanditReranker.fit); every
    # step ships the queries and their candidate id lists host -> device (each query's candidates in a
    # shuffled order), streams the candidates out of the corpus, scores, selects Top-K and reads it back.
    if not args.no_e2e:
        from paper_2602_02827_b200.batch import Corpus

        _log("e2e through Corpus.rerank_topk")

        corpus = Corpus(batch.d_tokens, do)
        rng = np.random.default_rng(1234 + rank)
        cand = np.concatenate([qd[q] + rng.permutation(int(qd[q + 1] - qd[q])) for q in range(nq)]).astype(np.int64)
        cand_t = torch.from_numpy(cand).pin_memory()
        q_host = batch.q_tokens.cpu().pin_memory()
        for _ in range(2):
            corpus.rerank_topk(q_host, qo, cand_t, qd, K)
        torch.cuda.synchronize()
        _barrier()
        e_steps = max(3, args.steps)
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e_steps):
            oi, ov = corpus.rerank_topk(q_host, qo, cand_t, qd, K)
        e1.record(stream)
        torch.cuda.synchronize()
        wall_ms = (time.perf_counter() - t0) * 1e3 / e_steps
        e_ms, = _reduce([max(e0.elapsed_time(e1) / e_steps, wall_ms)])
        h2d, = _reduce([q_host.numel() * q_host.element_size() + cand.nbytes + 2 * 8 * (nq + 1)], "sum")
        if rank == 0:
            got_docs = np.take_along_axis(cand.reshape(nq, -1), oi.numpy().astype(np.int64), axis=1) \
                if np.all(np.diff(qd) == qd[1] - qd[0]) else None
            ref_docs = idx.cpu().numpy().astype(np.int64) + qd[:-1, None]
            result["e2e"] = {"value": cells_total / (e_ms / 1e3), "unit": UNIT,
                             "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(nq_all * K * 8),
                             "ms_per_step": e_ms,
                             "api": "batch.Corpus.rerank_topk: corpus resident in HBM (fit once, untimed); per step "
                                    "H2D query tokens + candidate ids, maxsim_docs_kernel scores the candidates in "
                                    "place in the corpus (document tiles by TMA, tcgen05), Top-K, D2H Top-K; "
                                    "max of device-event and host wall time, max over ranks",
                             "topk_equals_device_path": bool(got_docs is not None and
                                                             np.array_equal(got_docs, ref_docs))}
        del corpus
        # cold variant: every document token crosses PCIe each step (no resident corpus)
        hb = HostBatch.from_device_batch(batch)
        out = (torch.empty((nq, K), dtype=torch.int32).pin_memory(), torch.empty((nq, K)).pin_memory())
        rerank_topk_host(hb, K, out=out)
        torch.cuda.synchronize()
        _barrier()
        e0.record(stream)
        for _ in range(2):
            rerank_topk_host(hb, K, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
        cold_ms, = _reduce([e0.elapsed_time(e1) / 2])
        cold_h2d, = _reduce([hb.h2d_bytes], "sum")
        if rank == 0:
            result["e2e_cold"] = {"value": cells_total / (cold_ms / 1e3), "unit": UNIT,
                                  "h2d_bytes_per_step": int(cold_h2d), "d2h_bytes_per_step": int(nq_all * K * 8),
                                  "ms_per_step": cold_ms,
                                  "api": "batch.rerank_topk_host: all doc tokens H2D every step (PCIe bound)"}
        del hb

    # ------------------------------------------------ the sections below are reported beside the headline;
    # a failure in one is recorded, not fatal (every rank runs the same code on the same shapes, so a
    # failure is symmetric across ranks)
    def section(name, fn):
        elapsed, = _reduce([time.perf_counter() - _T0])  # max over ranks: the same decision everywhere
        if elapsed >= args.budget_s:
            _log(f"section {name}: skipped (past the --budget-s {args.budget_s:.0f} s time budget)")
            if rank == 0:
                result[name] = {"skipped": f"time budget of {args.budget_s:.0f} s used up by the earlier sections"}
            return
        _log(f"section {name}: start")
        # multi-rank sections exchange data between ranks inside kernels and collectives: if a peer is lost, a
        # rank can wait forever. A watchdog then prints the line with what is already measured and ends the rank.
        timer = None
        if world > 1:
            def _bail():
                if rank == 0:
                    result[name] = {"error": f"watchdog: section did not finish within {args.section_timeout_s:.0f} s"}
                    print(json.dumps(result), flush=True)
                os._exit(0)

            timer = threading.Timer(args.section_timeout_s, _bail)
            timer.daemon = True
            timer.start()
        try:
            out = fn()
        except Exception as e:  # noqa: BLE001
            out = {"error": f"{type(e).__name__}: {e}"[:500]}
            print(f"bench: section {name} failed: {out['error']}", file=sys.stderr, flush=True)
        finally:
            if timer is not None:
                timer.cancel()
        _log(f"section {name}: done")
        if rank == 0:
            result[name] = out

    if not args.no_bandit:
        section("bandit", lambda: run_bandit(args, batch, host_off, cfg, rank, world, qa))
    del batch
    torch.cuda.empty_cache()
    if not args.no_p1_sharded:
        section("p1_sharded", lambda: run_p1_sharded(args, rank, world))
        torch.cuda.empty_cache()
    if not args.no_drop_in:
        section("drop_in", lambda: run_drop_in(args, rank, world))
    if not args.no_stage1:
        section("stage1", lambda: run_stage1(args, rank, world))
    if not args.no_p2_sharded:
        torch.cuda.empty_cache()
        section("bandit_sharded", lambda: run_p2_sharded(args, rank, world))
    _log("done")
    if rank == 0:
        print(json.dumps(result), flush=True)


def run_p1_sharded(args, rank, world):
    """cfg4 (one query, 100k candidates) exhaustive Top-100, documents sharded over the ranks:
    rank r scores its token-balanced contiguous document range with the tcgen05 scorer, takes its local
    Top-100 on the device, and ONE all-gather of 100 (score, global id) pairs per rank (NCCL over NVLink)
    feeds a device Top-K merge over the gathered lists, which ranks by (-score, id) exactly like the 1-GPU
    Top-K (rank-major gather order = id order for equal scores). Rank 0 checks the merged list against the
    single-GPU Top-100 of the whole pool."""
    import numpy as np
    import torch

    from paper_2602_02827_b200 import workloads as W
    from paper_2602_02827_b200.batch import TokenBatch, maxsim_scores, topk
    from paper_2602_02827_b200.dist import balanced_ranges

    cfg = W.CONFIGS["cfg4"]
    K = cfg.k
    b, (qo, do, qd) = W.gen_batch_device(cfg, n_queries=1, seed=0)  # the same pool on every rank
    N = b.n_docs
    single = None
    if rank == 0:
        s_all = maxsim_scores(b)
        single = topk(s_all, b.q_doc_off, K, N)[0].cpu().numpy().ravel().tolist()
        del s_all
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import maxsim_ref

        lim = _blas_one_thread()
        n_s = 5000
        q64 = b.q_tokens.double().cpu().numpy()
        toks = b.d_tokens[: int(do[n_s])].double().cpu().numpy()
        t0 = time.perf_counter()
        maxsim_ref.score_query(q64, [toks[do[i]:do[i + 1]] for i in range(n_s)], K)
        cpu_s = time.perf_counter() - t0
        del lim, toks
        T_ = int(qo[1] - qo[0])
        cpu = {"value": n_s * T_ / cpu_s, "unit": "cells/s", "cores": 1, "kind": "port",
               "full_query_s_extrapolated": cpu_s * N / n_s,
               "sample": f"oracle/maxsim_ref over the first {n_s} of the 100k documents ({cpu_s:.1f} s)"}
    lo, hi = balanced_ranges(do, world)[rank]
    local = (do[lo:hi + 1] - do[lo]).astype(np.int64)
    shard = b.d_tokens[int(do[lo]):int(do[hi])].clone()
    sb = TokenBatch.from_device(b.q_tokens, b.q_tok_off, shard, torch.from_numpy(local).cuda(),
                                torch.tensor([0, hi - lo], dtype=torch.int64, device="cuda"), False,
                                host_offsets=(qo, local, np.array([0, hi - lo], np.int64)))
    del b
    torch.cuda.empty_cache()
    dist = _dist()
    kk = min(K, hi - lo)
    scores = torch.empty(hi - lo, dtype=torch.float32, device="cuda")
    g_s = torch.empty(world * K, dtype=torch.float32, device="cuda")
    g_i = torch.empty(world * K, dtype=torch.int64, device="cuda")
    off_m = torch.tensor([0, world * K], dtype=torch.int64, device="cuda")

    def step():
        maxsim_scores(sb, out=scores)
        li, lv = topk(scores, sb.q_doc_off, kk, hi - lo)
        s = torch.full((K,), float("-inf"), dtype=torch.float32, device="cuda")
        i = torch.full((K,), -1, dtype=torch.int64, device="cuda")
        s[:kk] = lv.view(-1)
        i[:kk] = li.view(-1).to(torch.int64) + lo
        if dist is not None:
            dist.all_gather_into_tensor(g_s, s)
            dist.all_gather_into_tensor(g_i, i)
        else:
            g_s.copy_(s)
            g_i.copy_(i)
        mi, mv = topk(g_s, off_m, K, world * K)
        return g_i[mi.view(-1).to(torch.int64)]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    _barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        ids = step()
    e1.record()
    torch.cuda.synchronize()
    ms, = _reduce([e0.elapsed_time(e1) / args.steps])
    merged = ids.cpu().numpy().tolist()
    if rank != 0:
        return None
    T = int(qo[1] - qo[0])
    return {"what": "cfg4 exhaustive Top-100 (one query, 100k docs, Lq=32, d=128, f16) document-sharded over "
                    f"{world} rank(s): per-rank tcgen05 scorer + local Top-100, one all-gather of 100 (score, id) "
                    "pairs per rank, device Top-K merge by (-score, id)",
            "ranks": world, "ms": ms, "cells_per_s": N * T / (ms / 1e3),
            "doc_tokens_rank0": int(local[-1]), "exchange_bytes_per_rank": K * 12,
            "topk_equal_single_gpu": merged == single, "cpu_baseline": cpu,
            "gpu_launches": 3 + (2 if world > 1 else 0)}


def run_p2_sharded(args, rank, world):
    """cfg4 (one query, 100k candidates) Col-Bandit with the documents split over the ranks: each rank holds
    its shard's tokens and keeps the replicated run state; the revealed value crosses to the other ranks
    every iteration. Two exchange paths: "mailbox" (sharded.run_mailbox: ONE persistent kernel per rank, the
    owner stores the cell into the peers' inboxes over NVLink peer memory) and "host_stepped" (sharded.drive:
    a step kernel + NCCL all-reduce MAX per iteration, 64 per CUDA graph). Rank 0 also runs the single-GPU
    kernel on the whole pool and checks that every trace is identical."""
    import numpy as np
    import torch

    from paper_2602_02827_b200 import BanditConfig, BanditJob, run_batch
    from paper_2602_02827_b200 import workloads as W
    from paper_2602_02827_b200.batch import TokenBatch
    from paper_2602_02827_b200.dist import balanced_ranges
    from paper_2602_02827_b200.sharded import ShardedBanditRun, allreduce_exchange, drive, run_mailbox

    cfg = W.CONFIGS["cfg4"]
    b, (qo, do, qd) = W.gen_batch_device(cfg, n_queries=1, seed=0)  # the same pool on every rank
    N, T = b.n_docs, int(qo[1] - qo[0])
    bc = BanditConfig(k=cfg.k, seed=(0, 0))
    lo, hi = balanced_ranges(do, world)[rank]
    local = np.zeros(N + 1, np.int64)
    local[lo:hi + 1] = do[lo:hi + 1] - do[lo]
    local[hi + 1:] = do[hi] - do[lo]
    shard_tokens = b.d_tokens[int(do[lo]):int(do[hi])].clone()
    sb = TokenBatch.from_device(b.q_tokens, b.q_tok_off, shard_tokens, torch.from_numpy(local).cuda(), b.q_doc_off,
                                False, host_offsets=(qo, local, qd))
    single = None
    if rank == 0:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        single = run_batch([BanditJob(bc, N, T, 0, 0, (-1.0, 1.0))], batch=b)[0]
        e1.record()
        torch.cuda.synchronize()
        single_ms = e0.elapsed_time(e1)
        cpu = None
        if world == 1 and not args.no_cpu:
            # the reference's loop on this exact pool: oracle/bandit_ref over the float64 cells (the device cell
            # kernel's cells are bit-equal to the reference's, tests/test_gpu_cfg4.py), trace checked live
            from oracle import bandit_ref
            from paper_2602_02827_b200.batch import exact_cells

            cells = exact_cells(b, with_scores=False)[0][:, :T].cpu().numpy()
            t0 = time.perf_counter()
            ref = bandit_ref.run(cells, -1.0, 1.0, cfg.k, seed=(0, 0), indexed=True)
            cpu_s = time.perf_counter() - t0
            cpu = {"loop_s": cpu_s, "revealed_cells_per_s": len(ref.reveals) / cpu_s, "cores": 1, "kind": "port",
                   "sample": "the whole cfg4 run: oracle/bandit_ref loop (indexed ranking: sorted key list + lazy heaps, "
                             "as bandit.py:249-284) over precomputed float64 cells (row "
                             "computation excluded: that is P1, see p1_sharded.cpu_baseline)",
                   "trace_equal_device": ref.reveals == single.reveals and ref.topk == single.topk}
            del cells
    del b
    torch.cuda.empty_cache()
    # ---- mailbox: one persistent launch per rank
    if world > 1:
        tm = {}
        res_m = run_mailbox(sb, (lo, hi), bc, timing=tm)
        mb_ms, = _reduce([tm["ms"]])
    else:
        from paper_2602_02827_b200.sharded import run_local_shards

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res_m = run_local_shards(sb, [(lo, hi)], bc)[0]
        e1.record()
        torch.cuda.synchronize()
        mb_ms = e0.elapsed_time(e1)
    # ---- host-stepped: step kernel + collective per iteration
    hs = None
    if not args.no_p2_host_stepped:
        exchange = allreduce_exchange() if world > 1 else (lambda x, n: None)
        run = ShardedBanditRun(sb, (lo, hi), bc)
        torch.cuda.synchronize()
        _barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res_h = drive(run, exchange)
        e1.record()
        torch.cuda.synchronize()
        hs_ms, = _reduce([e0.elapsed_time(e1)])
        hs = (res_h, hs_ms, run.steps)
    if rank != 0:
        return None
    lens = np.diff(do)
    gather = int(lens[res_m.reveals.i.astype(np.int64)].sum()) * 128 * 2
    hbm_peak, _, peak_kind = _peaks()
    out = {"what": "Col-Bandit run() on one cfg4 query (100k docs, Lq=32, d=128, f16, K=100), documents sharded "
                   f"over {world} rank(s) by token count; replicated run state; every revealed cell crosses to "
                   "the other ranks",
           "ranks": world, "iterations": res_m.iterations, "reveals": len(res_m.reveals),
           "single_gpu_persistent_ms": single_ms, "single_gpu_us_per_iteration": single_ms * 1e3 / single.iterations,
           "cpu_baseline": cpu,
           "mailbox": {"ms": mb_ms, "us_per_iteration": mb_ms * 1e3 / res_m.iterations,
                       "revealed_cells_per_s": len(res_m.reveals) / (mb_ms / 1e3),
                       "gather_frac_of_hbm_per_gpu": gather / world / (mb_ms / 1e3) / 1e9 / hbm_peak,
                       "trace_equal_single_gpu": res_m.reveals == single.reveals and res_m.topk == single.topk,
                       "exchange": "none (1 rank)" if world == 1 else
                       "owner stores (value, flag) into every peer's inbox over NVLink (CUDA IPC), release/acquire",
                       "gpu_launches": 1}}
    if hs is not None:
        res_h, hs_ms, steps = hs
        out["host_stepped"] = {"ms": hs_ms, "us_per_iteration": hs_ms * 1e3 / res_h.iterations,
                               "trace_equal_single_gpu": res_h.reveals == single.reveals and res_h.topk == single.topk,
                               "exchange": "none (1 rank)" if world == 1 else
                               "NCCL all-reduce MAX, 8 B per iteration, NVLink",
                               "gpu_launches": steps}
    return out


def run_drop_in(args, rank, world):
    """The reference-facing names on cfg2 queries, host arrays in, Python results out, validation included:
    ``MaxSimOracle(QueryTokens(q), [DocTokens(...) x 1000], Similarity("dot", -1, 1))`` (oracle.py:107-144),
    ``.exact_topk(10)`` (oracle.py:229-235) and ``run(oracle, CellBounds.uniform(...), BanditConfig(k=10,
    seed=(0, q)))`` (bandit.py:169) — per query, as a caller of the reference would use them — beside the
    reference algorithm on the same query (oracle port, one core) and a parity check of both outputs."""
    if rank != 0:
        return None
    import numpy as np

    from oracle import bandit_ref, maxsim_ref
    from paper_2602_02827_b200 import (BanditConfig, CellBounds, DocTokens, MaxSimOracle, QueryTokens, Similarity,
                                       run)
    from paper_2602_02827_b200 import workloads as W

    cfg = W.CONFIGS["cfg2"]
    n_q = 3
    t_build = t_topk = t_run = t_cpu_p1 = t_cpu_p2 = 0.0
    same = True
    lim = _blas_one_thread()
    for q in range(n_q + 1):  # query 0 warms up (untimed)
        case = W.gen_query(cfg, q)
        off = case.doc_offsets
        raw = [case.doc_tokens[off[i]:off[i + 1]] for i in range(case.n_docs)]
        t0 = time.perf_counter()
        oracle = MaxSimOracle(QueryTokens(case.query), [DocTokens(f"d{i}", x) for i, x in enumerate(raw)],
                              Similarity("dot", -1.0, 1.0))
        t1 = time.perf_counter()
        top = oracle.exact_topk(cfg.k)
        t2 = time.perf_counter()
        res = run(oracle, CellBounds.uniform(case.n_docs, 32, -1.0, 1.0), BanditConfig(k=cfg.k, seed=(0, q)))
        t3 = time.perf_counter()
        q64, d64 = case.query64(), case.docs64()
        t4 = time.perf_counter()
        ref_s, ref_top, cells = maxsim_ref.score_query(q64, d64, cfg.k)
        t5 = time.perf_counter()
        ref = bandit_ref.run(maxsim_ref.cell_matrix(q64, d64), -1.0, 1.0, cfg.k, seed=(0, q))
        t6 = time.perf_counter()
        same &= top == list(ref_top) and res.reveals == ref.reveals and res.topk == ref.topk
        if q:
            t_build += t1 - t0
            t_topk += t2 - t1
            t_run += t3 - t2
            t_cpu_p1 += t5 - t4
            t_cpu_p2 += t6 - t5
    del lim
    return {"what": "reference-facing API per cfg2 query (1000 fp16 docs from host numpy arrays): MaxSimOracle "
                    "construction (validation, float64 view, H2D), exact_topk(10), run(oracle, generic bounds, "
                    "BanditConfig(k=10, seed=(0, q))); beside the reference algorithm (oracle port, 1 core)",
            "queries": n_q, "construct_ms": t_build * 1e3 / n_q, "exact_topk_ms": t_topk * 1e3 / n_q,
            "run_ms": t_run * 1e3 / n_q,
            "cpu_reference": {"exact_topk_ms": t_cpu_p1 * 1e3 / n_q, "run_ms": t_cpu_p2 * 1e3 / n_q, "cores": 1,
                              "kind": "port"},
            "outputs_equal_reference_algorithm": bool(same), "gpu_launches": 4}


def run_stage1(args, rank, world):
    """Stage-1 scan (generate_candidates) of one cfg4 query over the 100k-document corpus, then the full
    ColBanditReranker.rerank through the public API (Stage 1 + ANN bounds + device bandit)."""
    import ctypes

    import numpy as np
    import torch

    from paper_2602_02827_b200 import _lib
    from paper_2602_02827_b200 import workloads as W
    from paper_2602_02827_b200.batch import Corpus, dtype_code
    from paper_2602_02827_b200.pipeline import stage1_topk
    from paper_2602_02827_b200.reranker import ColBanditReranker

    cfg = W.CONFIGS["cfg4"]
    b4, (qo, do, qd) = W.gen_batch_device(cfg, n_queries=1, seed=rank)
    corpus = Corpus(b4.d_tokens, do, clamp_negative=True)
    q = b4.q_tokens
    kp, R, T = 10, int(q.shape[0]), corpus.n_tokens
    lib = _lib.load()
    s = _lib.CbxBatch()
    s.q_tokens, s.n_q_tokens = q.data_ptr(), R
    s.d_tokens, s.n_d_tokens = corpus.tokens.data_ptr(), T
    s.dim, s.dtype, s.clamp_negative, s.max_lq = corpus.dim, dtype_code(q.dtype), 1, R
    wsb = lib.cbx_stage1_workspace_bytes(ctypes.byref(s), kp, _lib.CBX_PATH_TC)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    tok = torch.empty((R, kp), dtype=torch.int64, device="cuda")
    val = torch.empty((R, kp), dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    norm = corpus.norm_max()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def call():
        _lib.check(lib.cbx_stage1_topk(ctypes.byref(s), kp, _lib.CBX_PATH_TC, ctypes.c_float(norm), tok.data_ptr(),
                                       val.data_ptr(), st.data_ptr(), ws.data_ptr(), wsb, stream), "stage1")

    for _ in range(args.warmup):
        call()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        call()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    tc_status = int(st.item())
    tok_tc, val_tc = tok.cpu().numpy(), val.cpu().numpy()
    tok_sx, val_sx = stage1_topk(corpus, q, kp, True, path="simt")
    hbm_peak, _, peak_kind = _peaks()
    nbytes = T * corpus.dim * corpus.tokens.element_size()
    # the facade end to end: host query in, Top-K doc ids out (Stage 1 + pool gather + ANN bounds + bandit)
    est = ColBanditReranker(k=10, k_prime=kp, similarity="dot", clamp_negative=True).fit(corpus)
    qh = q.cpu()
    est.rerank(qh, query_index=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        o = est.rerank(qh, query_index=0)
    facade_ms = (time.perf_counter() - t0) * 1e3 / reps
    if rank != 0:
        return None
    out = {"what": "pipeline.generate_candidates Stage-1 scan (cbx_stage1_topk, tcgen05 + float64 refine): one cfg4 "
                   f"query ({R} tokens) against the 100k-doc cfg4 corpus ({T} tokens, d={corpus.dim}, "
                   f"{cfg.dtype}), k'={kp}, clamp_negative",
           "ms": ms, "sims_per_s": R * T / (ms / 1e3),
           "roofline": {"bound": "hbm", "kernel": "stage1_scan_kernel (+ pre-pass, seed, refine)",
                        "achieved": nbytes / (ms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                        "frac": nbytes / (ms / 1e3) / 1e9 / hbm_peak, "peak_kind": peak_kind,
                        "alg_bytes_per_call": nbytes},
           "parity": {"tc_equals_float64_simt_scan": bool(np.array_equal(tok_tc, tok_sx) and
                                                          np.array_equal(val_tc, val_sx)),
                      "tc_status": tc_status},
           "facade": {"api": "ColBanditReranker(k=10, k_prime=10, similarity='dot').fit(Corpus).rerank(query)",
                      "ms_per_query": facade_ms, "candidates": len(o.candidates), "coverage": o.coverage,
                      "terminated_by": o.result.terminated_by},
           "gpu_launches": 5}
    if world == 1 and not args.no_cpu:
        from oracle import stage1_ref

        lim = _blas_one_thread()
        n_docs = 1500
        q64 = q.double().cpu().numpy()
        toks = corpus.tokens[: int(do[n_docs])].double().cpu().numpy()
        docs = [toks[do[i]:do[i + 1]] for i in range(n_docs)]
        t0 = time.perf_counter()
        _, _, ref_nb = stage1_ref.generate_candidates(q64, docs, kp, True)
        cpu_s = time.perf_counter() - t0
        del lim
        # the device scan (tcgen05 filter + float64 refine) over the same sub-corpus against the CPU oracle's
        # neighbour lists: global token index and float64 similarity, token for token
        sub = Corpus(corpus.tokens[: int(do[n_docs])], do[: n_docs + 1].copy(), clamp_negative=True)
        tk_s, vl_s = stage1_topk(sub, q, kp, True, path="tc")
        ref_tok = np.array([[int(do[d]) + j for d, j, _ in nbs] for nbs in ref_nb], dtype=np.int64)
        ref_val = np.array([[v for *_, v in nbs] for nbs in ref_nb], dtype=np.float64)
        out["parity"]["tc_equals_cpu_oracle"] = bool(np.array_equal(tk_s, ref_tok) and np.array_equal(vl_s, ref_val))
        out["parity"]["cpu_oracle_sample"] = f"first {n_docs} cfg4 docs ({int(do[n_docs])} tokens), path " + \
            "/".join(sorted(set(stage1_topk.last_paths)))
        out["cpu_baseline"] = {"value": R * int(do[n_docs]) / cpu_s, "unit": "similarities/s", "cores": 1,
                               "kind": "port", "sample": f"oracle/stage1_ref.generate_candidates over the first "
                                                         f"{n_docs} cfg4 docs ({int(do[n_docs])} tokens), {cpu_s:.1f} s"}
    return out


def _bandit_traffic(name):
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    return json.load(open(tpath)).get(f"bandit_{name}") if os.path.exists(tpath) else None


def run_bandit(args, batch, host_off, cfg, rank, world, qa=0):
    """The Col-Bandit loop on this rank's query block (one CTA per run), timed on the device; the job's
    totals (runs, reveals, gathered bytes) are summed over the ranks and the time is the max over ranks."""
    import numpy as np
    import torch

    from paper_2602_02827_b200 import BanditConfig, BanditJob, run_batch
    from paper_2602_02827_b200.bandit import collect, launch_batch, prepare_batch

    qo, do, qd = host_off
    nq = batch.n_queries
    # seeds follow the reference's (random_state, query_index) convention with the GLOBAL query index
    jobs = [BanditJob(BanditConfig(k=cfg.k, seed=(0, qa + q)), int(qd[q + 1] - qd[q]), int(qo[q + 1] - qo[q]), q,
                      int(qd[q]), (-1.0, 1.0)) for q in range(nq)]
    lens = np.diff(do)
    elem = batch.d_tokens.element_size()
    # device time: descriptors prepared once (host seeding, H2D), then the launches alone are timed
    prep = prepare_batch(jobs, batch=batch)
    for _ in range(max(1, min(args.warmup, 2))):
        collect(launch_batch(prep), jobs, list(prep["results"]), return_traces=False)
    torch.cuda.synchronize()
    _barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    raw = launch_batch(prep)
    e1.record()
    torch.cuda.synchronize()
    ms, = _reduce([e0.elapsed_time(e1)])
    res = collect(raw, jobs, list(prep["results"]))
    # end to end through the public call (host seeding + descriptors + launches + traces back)
    _barrier()
    t0 = time.perf_counter()
    res_e2e = run_batch(jobs, batch=batch)
    e2e_ms, = _reduce([(time.perf_counter() - t0) * 1e3])
    assert all(a.reveals == b.reveals for a, b in zip(res_e2e, res))
    reveals = sum(len(r.reveals) for r in res)
    gather = 0
    for j, r in zip(jobs, res):
        if len(r.reveals):
            gather += int(lens[r.reveals.i.astype(np.int64) + j.row_begin].sum()) * batch.dim * elem
    cov = np.array([r.coverage for r in res])
    runs_all, reveals_all, gather_all, iters_all, cov_sum = _reduce(
        [len(jobs), reveals, gather, sum(r.iterations for r in res), cov.sum()], "sum")
    cov_min, = _reduce([-cov.min()])
    cov_max, = _reduce([cov.max()])
    if rank != 0:
        return None
    hbm_peak, _, peak_kind = _peaks()
    out = {"what": "Col-Bandit run() per query (one CTA each), BanditConfig defaults, generic bounds (-1, 1), "
                   "seed (0, q); queries sharded over the ranks like the headline",
           "runs": int(runs_all), "ms": ms, "queries_per_s": runs_all / (ms / 1e3),
           "revealed_cells_per_s": reveals_all / (ms / 1e3),
           "iterations": int(iters_all),
           "coverage_mean": cov_sum / runs_all, "coverage_min": -cov_min, "coverage_max": cov_max,
           "roofline": {"bound": "hbm (gather)", "achieved": gather_all / (ms / 1e3) / 1e9 / world,
                        "peak": hbm_peak, "unit": "GB/s per GPU",
                        "frac": gather_all / (ms / 1e3) / 1e9 / world / hbm_peak, "peak_kind": peak_kind,
                        "alg_bytes": int(gather_all),
                        "note": "algorithmic gather = sum over reveals of L_i*d*s (warm-up included); repeated "
                                "boundary rows hit L2/L1, so this can exceed DRAM traffic",
                        "traffic": _bandit_traffic(cfg.name) if world == 1 else None,
                        "traffic_note": "dram__bytes_read+write of one bandit_kernel launch on this config from "
                                        "the committed ncu capture (profiles/)"},
           "gpu_launches": 1 + (2 if prep["n_prewarm"] else 0),
           "e2e": {"ms": e2e_ms, "revealed_cells_per_s": reveals_all / (e2e_ms / 1e3),
                   "ratio_to_device": e2e_ms / ms,
                   "api": "bandit.run_batch(jobs, batch): host seeding + descriptors + launch + compacted trace "
                          "D2H (RunResult.reveals as numpy-backed Reveals)"}}
    # ---- the row-cache variant, accounted separately: once two cells of a row are revealed, the
    # next reveal computes all Lq cells of the row from one gather (the reference's oracle computes whole rows
    # on first touch, oracle.py:205-215), later reveals of the row are reads; same traces, fewer gathered
    # bytes, Lq x the tensor-core work per gather
    if world == 1:
        try:
            prep_rc = prepare_batch(jobs, batch=batch, row_cache=True)
            collect(launch_batch(prep_rc), jobs, list(prep_rc["results"]), return_traces=False)
            torch.cuda.synchronize()
            e0.record()
            raw_rc = launch_batch(prep_rc)
            e1.record()
            torch.cuda.synchronize()
            st = {}
            res_rc = collect(raw_rc, jobs, list(prep_rc["results"]), stats=st)
            g_on = g_fill = fills = 0
            thr = 2  # run_batch(row_cache=True): a reveal fills its row once two of the row's cells are revealed
            for j, r in zip(jobs, res_rc):
                cnt = np.bincount(r.reveals.i.astype(np.int64), minlength=j.n_rows)
                L = lens[j.row_begin:j.row_begin + j.n_rows]
                g_on += int((L * np.minimum(cnt, thr)).sum())  # single-cell gathers (warm-up + first adaptive)
                fills += int((cnt > thr).sum())
                g_fill += int(L[cnt > thr].sum())              # one whole-row gather each
            out["row_cache"] = {
                "what": "run_batch(..., row_cache=True): the reveal that finds two cells of its row revealed computes all "
                        "Lq cells of the row from one gather, later reveals of the row read them back; reported "
                        "beside, not instead of, the on-demand loop",
                "ms": e0.elapsed_time(e1), "revealed_cells_per_s": reveals / (e0.elapsed_time(e1) / 1e3),
                "trace_identical_to_on_demand": all(a.reveals == b.reveals and a.topk == b.topk
                                                    for a, b in zip(res_rc, res)),
                "rows_filled": int(st["rows_filled"].sum()), "rows_filled_from_traces": int(fills),
                "reveals_served_from_cache": int(reveals - sum(int(np.minimum(np.bincount(
                    r.reveals.i.astype(np.int64), minlength=j.n_rows), thr + 1).sum()) for j, r in zip(jobs, res_rc))),
                "gather_bytes": {"single_cell_reveals": g_on * batch.dim * elem,
                                 "row_fills": g_fill * batch.dim * elem,
                                 "on_demand_loop_total": int(gather)},
                "cells_computed_per_fill": "Lq (all columns of the row)"}
        except Exception as e:  # noqa: BLE001
            out["row_cache"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    # parity + CPU baseline on sampled queries: the oracle loop must reproduce the device trace
    from oracle import bandit_ref, maxsim_ref

    lim = _blas_one_thread()
    n_chk, same, cpu_s, cpu_rev, cov_err = 0, True, 0.0, 0, 0.0
    for q in range(nq):
        qt, docs = _query_host(batch, host_off, q)
        t0 = time.perf_counter()
        cells = maxsim_ref.cell_matrix(qt, docs)
        ref = bandit_ref.run(cells, -1.0, 1.0, cfg.k, seed=(0, qa + q))
        cpu_s += time.perf_counter() - t0
        cpu_rev += len(ref.reveals)
        same &= (res[q].reveals == ref.reveals and ref.topk == res[q].topk)
        cov_err = max(cov_err, abs(ref.coverage - res[q].coverage))
        n_chk += 1
        if n_chk >= args.check_queries and cpu_s >= args.cpu_seconds / 2:
            break
    del lim
    out["parity"] = {"queries_checked": n_chk, "trace_identical": bool(same), "coverage_abs_err_max": cov_err}
    if world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        _log(f"bandit: CPU baseline on {cores} cores (spawned workers)")
        bwall, bouts = cpu_pool(cfg.name, cores, _ref_bandit_task, reps=1)
        out["cpu_baseline"] = {"value": sum(r for _, r in bouts) / bwall, "unit": "revealed cells/s", "cores": cores,
                               "kind": "port", "queries_per_s": cores / bwall,
                               "sample": f"{cores} {cfg.name} Col-Bandit runs, one per process on every host core "
                                         f"(rows + oracle/bandit_ref loop), {bwall:.1f} s wall",
                               "one_core": {"value": cpu_rev / cpu_s, "queries_per_s": n_chk / cpu_s,
                                            "sample": f"{n_chk} of this batch's queries, {cpu_s:.1f} s"}}
    return out


# ---------------------------------------------------------------------------- reference arm
_REF_STATE = {}


def _ref_init(cfg_name, worker_seed):
    from threadpoolctl import threadpool_limits

    from paper_2602_02827_b200 import workloads as W

    threadpool_limits(1)
    case = W.gen_query(cfg_name, worker_seed)
    _REF_STATE["case"] = (case.query64(), case.docs64(), W.CONFIGS[cfg_name].k)


def _ref_task(_):
    """P1 of one query through the reference algorithm (oracle port): float64 cells, fsum scores, lexsort."""
    from oracle import maxsim_ref

    q, docs, k = _REF_STATE["case"]
    t0 = time.perf_counter()
    maxsim_ref.score_query(q, docs, k)
    return time.perf_counter() - t0, len(docs) * q.shape[0]


def _ref_bandit_task(q_index):
    """P2 of one query through the reference algorithm: the rows it touches (all of them: the warm-up reveals
    every row, oracle.py:205-215) + the loop (bandit_ref restates bandit.py:169-350), seed (0, q)."""
    from oracle import bandit_ref, maxsim_ref

    q, docs, k = _REF_STATE["case"]
    t0 = time.perf_counter()
    cells = maxsim_ref.cell_matrix(q, docs)
    res = bandit_ref.run(cells, -1.0, 1.0, k, seed=(0, q_index))
    return time.perf_counter() - t0, len(res.reveals)


def cpu_pool(cfg_name, workers, fn, reps=1, timeout_s=240.0):
    """Run fn once per worker per rep in a process pool whose workers hold one query of the config; returns
    (wall seconds of the timed maps, summed per-task results). A process that has initialised CUDA must not
    fork (the children inherit the driver's and OpenMP's locked state and can hang): it spawns fresh
    interpreters instead; every map is bounded by ``timeout_s``."""
    import concurrent.futures as cf
    import multiprocessing as mp

    cuda_up = False
    if "torch" in sys.modules:
        import torch

        cuda_up = torch.cuda.is_initialized()
    ctx = mp.get_context("spawn" if cuda_up else "fork")
    ex = cf.ProcessPoolExecutor(workers, mp_context=ctx, initializer=_ref_init, initargs=(cfg_name, 0))
    try:
        list(ex.map(_noop, range(workers), timeout=timeout_s))  # initialise every worker (untimed)
        t0 = time.perf_counter()
        out = []
        for _ in range(reps):
            out += list(ex.map(fn, range(workers), timeout=timeout_s))
        wall = time.perf_counter() - t0
    except BaseException:
        for pr in list(getattr(ex, "_processes", {}).values()):  # a stuck worker must not outlive the bench
            pr.kill()
        ex.shutdown(wait=False, cancel_futures=True)
        raise
    ex.shutdown()
    return wall, out


def _noop(_):
    time.sleep(0.05)
    return 0


def run_reference(args):
    from paper_2602_02827_b200 import workloads as W

    cfg = W.CONFIGS[args.config]
    cores = os.cpu_count() or 1
    workers = max(1, min(cores, args.ref_workers or cores))
    # each worker generates one query of the config once (untimed), then scores it once per step
    cpu_pool(cfg.name, workers, _ref_task, reps=args.warmup)
    wall, outs = cpu_pool(cfg.name, workers, _ref_task, reps=args.steps)
    cells = sum(c for _, c in outs)
    value = cells / wall
    # the Col-Bandit loop on the same cores (one run per worker, bounded)
    bwall, bouts = cpu_pool(cfg.name, workers, _ref_bandit_task, reps=1)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype,
        "data": "synthetic (numpy, BASELINE.json configs[1] recipe)",
        "config": {"workload": f"{cfg.name}: {cfg.n_docs} docs/query, Lq={cfg.lq[0]}, d={cfg.dim}, {cfg.dtype}, "
                               f"K={cfg.k}", "queries_per_step": workers},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": f"{workers} {cfg.name} queries per step, one per process (ProcessPoolExecutor, "
                                   f"BLAS 1 thread each; oracle/maxsim_ref)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "bandit": {"revealed_cells_per_s": sum(r for _, r in bouts) / bwall, "queries_per_s": workers / bwall,
                   "cores": workers, "kind": "port",
                   "sample": f"{workers} {cfg.name} Col-Bandit runs (rows + oracle/bandit_ref loop), one per process"},
    }), flush=True)


def run_dry(args, rank, world):
    """--dry-run: the multi-rank plumbing without a GPU (gloo): the query plan, this rank's block, a
    host-side stand-in step timed per rank, the max-over-ranks time and the JSON line of rank 0."""
    import numpy as np

    from paper_2602_02827_b200 import workloads as W

    cfg, lens_all, lqs_all = W.batch_plan(args.config, args.queries, seed=0)
    blocks = W.query_blocks(lens_all, world)
    qa, qb = blocks[rank]
    _barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        tok = int(lens_all[qa:qb].sum())  # stand-in for scoring the block: its doc-token count
    ms, = _reduce([(time.perf_counter() - t0) * 1e3 / args.steps])
    tok_all, nq_all = _reduce([tok, qb - qa], "sum")
    if rank == 0:
        cells = int(lens_all.shape[1] * lqs_all.sum())
        print(json.dumps({"metric": METRIC, "value": cells / max(ms, 1e-9) * 1e3, "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                          "scaling": "strong", "dry_run": True, "dtype": cfg.dtype,
                          "config": {"workload": cfg.name, "queries": int(nq_all), "query_blocks": blocks,
                                     "doc_tokens": int(tok_all)}}), flush=True)


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _spawned(local_rank, args, world, port):
    """Entry of a rank spawned by ``bench.py --gpus N`` (no torchrun): the torchrun environment by hand."""
    os.environ.update({"RANK": str(local_rank), "LOCAL_RANK": str(local_rank), "WORLD_SIZE": str(world),
                       "LOCAL_WORLD_SIZE": str(world), "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    _rank_main(args)


def _rank_main(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        # the reference's CPU algorithm runs once, on rank 0; other ranks exit without work
        if rank == 0:
            run_reference(args)
        return
    if args.gpus != world and world > 1:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        import torch
        import torch.distributed as dist

        if args.dry_run:
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.dry_run:
            run_dry(args, rank, world)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--queries", type=int, default=None)
    ap.add_argument("--check-queries", type=int, default=4)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-workers", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-bandit", action="store_true")
    ap.add_argument("--no-p1-sharded", action="store_true")
    ap.add_argument("--no-stage1", action="store_true")
    ap.add_argument("--no-drop-in", action="store_true")
    ap.add_argument("--no-p2-sharded", action="store_true")
    ap.add_argument("--no-p2-host-stepped", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="launcher/sharding/reduction only, no GPU (gloo)")
    ap.add_argument("--section-timeout-s", type=float, default=240.0,
                    help="multi-rank runs: a section beside the headline that takes longer ends the run with the "
                         "line measured so far")
    ap.add_argument("--budget-s", type=float, default=420.0,
                    help="sections beside the headline start only while the run is younger than this (seconds)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        # no torchrun: spawn one process per GPU here (torchrun's environment, 127.0.0.1 rendezvous)
        import torch.multiprocessing as tmp

        tmp.start_processes(_spawned, args=(args, args.gpus, _free_port()), nprocs=args.gpus, join=True,
                            start_method="spawn")
        return
    _rank_main(args)


if __name__ == "__main__":
    main()
