#!/usr/bin/env python
"""Benchmark of the exhaustive MaxSim reranker (P1) — the driver's contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

One "step" = one pass of the hot path over one batch: MaxSim scores of every
candidate of every query (tcgen05 dense scorer) + per-query Top-K. The
workload is BASELINE.json configs[1] ("cfg2": 256 queries x 1000 candidates,
Lq = 32, d = 128, fp16, lognormal doc lengths, K = 10), drawn on the device
(synthetic, seeded by rank). Inputs (11.7 GB of doc tokens) are larger than
L2 (126 MB), so no flush is needed between steps.

metric: MaxSim cells/s (cell = one (document, query token) pair), plus
queries/s and the scorer's achieved HBM GB/s against the measured peak.
Multi-GPU: one process per GPU, each with its own batch (weak scaling, no
collective on the data path); value = all ranks' cells / max-over-ranks time.

``--impl reference`` times the CPU oracle port (oracle/maxsim_ref — the
reference's float64 GEMM + column max + math.fsum + lexsort, restated) on
the box's host cores with one process per core, for the same metric/config.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MaxSim cells/sec (exhaustive rerank, oracle-matching Top-K)"
UNIT = "cells/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        import statistics

        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2602_02827_b200 import _lib
    from paper_2602_02827_b200 import workloads as W
    from paper_2602_02827_b200.batch import HostBatch, maxsim_scores, rerank_topk, rerank_topk_host, topk

    torch.cuda.set_device(local_rank)
    cfg = W.CONFIGS[args.config]
    batch, host_off = W.gen_batch_device(cfg, n_queries=args.queries, seed=rank)
    torch.cuda.synchronize()
    nq, K = batch.n_queries, cfg.k
    elem = batch.d_tokens.element_size()
    qo, do, qd = host_off
    cells_per_step = int(sum((qd[q + 1] - qd[q]) * (qo[q + 1] - qo[q]) for q in range(nq)))
    alg_bytes = int(batch.d_tokens.numel() * elem + batch.q_tokens.numel() * elem + 4 * batch.n_docs)
    alg_flops = int(2 * sum((do[qd[q + 1]] - do[qd[q]]) * (qo[q + 1] - qo[q]) for q in range(nq)) * batch.dim)

    stream = torch.cuda.current_stream()
    scores = torch.empty(batch.n_docs, dtype=torch.float32, device="cuda")

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        maxsim_scores(batch, out=scores)
        if ev is not None:
            ev[1].record(stream)
        idx, val = topk(scores, batch.q_doc_off, K, batch.max_q_docs)
        if ev is not None:
            ev[2].record(stream)
        return idx, val

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        start.record(stream)
        for i in range(args.steps):
            idx, val = step(evs[i])
        stop.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = start.elapsed_time(stop)
    kern_ms = [e[0].elapsed_time(e[1]) for e in evs]
    topk_ms = [e[1].elapsed_time(e[2]) for e in evs]
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(t.item())
    hbm_peak, tf_peak, peak_kind = _peaks()

    result = None
    if rank == 0:
        ms_step = ms_max / args.steps
        value = cells_per_step * world / (ms_step / 1e3)
        kavg = sum(kern_ms) / len(kern_ms)
        achieved = alg_bytes / (kavg / 1e3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            traffic = json.load(open(tpath)).get(args.config)
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic (device RNG, BASELINE.json configs[1] recipe)",
            "config": {"workload": f"{cfg.name}: {nq} queries x {cfg.n_docs} docs, Lq={cfg.lq[0]}, d={cfg.dim}, "
                                   f"lognormal lengths (mean 180, sigma 0.5, clip [16,512]), K={K}",
                       "queries_per_gpu": nq, "doc_tokens_per_gpu": int(batch.d_tokens.shape[0]),
                       "l2": "inputs (%.1f GB) exceed L2; no flush" % (alg_bytes / 1e9),
                       "parallelism": f"query-sharded x{world} (no collective)"},
            "queries_per_s": nq * world / (ms_step / 1e3),
            "scorer_ms": kavg, "topk_ms": sum(topk_ms) / len(topk_ms),
            "roofline": {"bound": "hbm", "kernel": "maxsim_tc_kernel", "achieved": achieved, "peak": hbm_peak,
                         "unit": "GB/s", "frac": achieved / hbm_peak, "peak_kind": peak_kind,
                         "alg_bytes_per_launch": alg_bytes, "traffic": traffic,
                         "tensor_tflops": alg_flops / (kavg / 1e3) / 1e12, "tensor_peak": tf_peak},
            "clocks": clocks.summary(),
            "gpu_launches": args.steps * 2,
        }

    # ------------------------------------------------ parity on a sample + CPU baseline (rank 0, N = 1)
    if rank == 0:
        from oracle import maxsim_ref

        n_check = min(nq, args.check_queries)
        idx_h = idx.cpu().numpy()
        sc_h = scores.cpu().numpy()
        ok = True
        cpu_cells, cpu_s = 0, 0.0
        try:
            from threadpoolctl import threadpool_limits
            lim = threadpool_limits(1)
        except Exception:
            lim = None
        for q in range(n_check):
            d0, d1 = int(qd[q]), int(qd[q + 1])
            qt = batch.q_tokens[int(qo[q]):int(qo[q + 1])].double().cpu().numpy()
            dt = batch.d_tokens[int(do[d0]):int(do[d1])].double().cpu().numpy()
            docs = [dt[int(do[i] - do[d0]):int(do[i + 1] - do[d0])] for i in range(d0, d1)]
            t0 = time.perf_counter()
            ref_s, ref_t, _ = maxsim_ref.score_query(qt, docs, K)
            cpu_s += time.perf_counter() - t0
            cpu_cells += (d1 - d0) * qt.shape[0]
            if not np.allclose(sc_h[d0:d1], ref_s, rtol=1e-3, atol=0):
                ok = False
            got = idx_h[q].tolist()
            if got != ref_t:
                for g_, r_ in zip(got, ref_t):
                    if g_ != r_ and abs(ref_s[g_] - ref_s[r_]) > 1e-3 * abs(ref_s[r_]):
                        ok = False
        if lim is not None:
            lim.unregister() if hasattr(lim, "unregister") else None
        result["parity"] = {"queries_checked": n_check, "scores_rtol": 1e-3, "topk_match": ok}
        if world == 1 and not args.no_cpu:
            result["cpu_baseline"] = {"value": cpu_cells / cpu_s, "unit": UNIT, "cores": 1, "kind": "port",
                                      "sample": f"{n_check} cfg2 queries (oracle/maxsim_ref: float64 GEMM + max + "
                                                f"fsum + lexsort, OPENBLAS 1 thread), {cpu_s:.1f} s"}

    # ------------------------------------------------ end-to-end through the public host API
    if not args.no_e2e:
        hb = HostBatch.from_device_batch(batch)
        out = (torch.empty((nq, K), dtype=torch.int32).pin_memory(), torch.empty((nq, K)).pin_memory())
        for _ in range(2):
            rerank_topk_host(hb, K, out=out)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_steps = max(2, min(args.steps, 5))
        e0.record(stream)
        for _ in range(e_steps):
            rerank_topk_host(hb, K, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if world > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        if rank == 0:
            e_ms = float(t.item()) / e_steps
            result["e2e"] = {"value": cells_per_step * world / (e_ms / 1e3), "unit": UNIT,
                             "h2d_bytes_per_step": hb.h2d_bytes, "d2h_bytes_per_step": int(nq * K * 8),
                             "ms_per_step": e_ms}
            ok = out[0].numpy().tolist() == idx.cpu().numpy().tolist()
            result["e2e"]["topk_equals_device_path"] = bool(ok)
    if rank == 0:
        print(json.dumps(result), flush=True)


# ---------------------------------------------------------------------------- reference arm
_REF_STATE = {}


def _ref_init(cfg_name, worker_seed):
    from threadpoolctl import threadpool_limits

    from paper_2602_02827_b200 import workloads as W

    threadpool_limits(1)
    case = W.gen_query(cfg_name, worker_seed)
    _REF_STATE["case"] = (case.query64(), case.docs64(), W.CONFIGS[cfg_name].k)


def _ref_task(_):
    from oracle import maxsim_ref

    q, docs, k = _REF_STATE["case"]
    t0 = time.perf_counter()
    maxsim_ref.score_query(q, docs, k)
    return time.perf_counter() - t0, len(docs) * q.shape[0]


def run_reference(args):
    import concurrent.futures as cf
    import multiprocessing as mp

    from paper_2602_02827_b200 import workloads as W

    cfg = W.CONFIGS[args.config]
    cores = os.cpu_count() or 1
    workers = max(1, min(cores, args.ref_workers or cores))
    ctx = mp.get_context("fork")
    # each worker generates query 0 of the config once (untimed), then scores it once per step
    with cf.ProcessPoolExecutor(workers, mp_context=ctx, initializer=_ref_init, initargs=(cfg.name, 0)) as ex:
        for _ in range(args.warmup):
            list(ex.map(_ref_task, range(workers)))
        t0 = time.perf_counter()
        cells = 0
        for _ in range(args.steps):
            for _, c in ex.map(_ref_task, range(workers)):
                cells += c
        wall = time.perf_counter() - t0
    value = cells / wall
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype,
        "data": "synthetic (numpy, BASELINE.json configs[1] recipe)",
        "config": {"workload": f"{cfg.name}: {cfg.n_docs} docs/query, Lq={cfg.lq[0]}, d={cfg.dim}, K={cfg.k}",
                   "queries_per_step": workers},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": f"{workers} cfg2 queries per step, one per process (ProcessPoolExecutor, "
                                   f"OPENBLAS 1 thread each; oracle/maxsim_ref)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--queries", type=int, default=None)
    ap.add_argument("--check-queries", type=int, default=4)
    ap.add_argument("--ref-workers", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args)
        return
    if world > 1:
        import torch

        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl")
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch

            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
