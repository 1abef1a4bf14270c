"""Time the device Stage-1 scan (cbx_stage1_topk) on a large synthetic corpus.

    python tools/prof_stage1.py [--tokens 17900000] [--dim 128] [--queries 1] [--lq 32] [--kp 10] [--path tc]

Reports per call: ms, corpus GB/s (corpus bytes x row blocks / time, the
algorithmic traffic of the scan) and the dense-equivalent TFLOP/s.
"""

import argparse
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2602_02827_b200 import _lib  # noqa: E402
from paper_2602_02827_b200.batch import Corpus, dtype_code  # noqa: E402
from paper_2602_02827_b200.pipeline import stage1_topk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=17_900_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--queries", type=int, default=1)
    ap.add_argument("--lq", type=int, default=32)
    ap.add_argument("--kp", type=int, default=10)
    ap.add_argument("--path", default="tc")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--dtype", default="f16")
    ap.add_argument("--check", action="store_true", help="compare with the SIMT scan")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(0)
    tdt = torch.float16 if a.dtype == "f16" else torch.bfloat16
    x = torch.randn((a.tokens, a.dim), device="cuda", generator=g)
    x = (x / x.norm(dim=1, keepdim=True)).to(tdt)
    lens = np.full(a.tokens // 180, 180, np.int64)
    lens[-1] += a.tokens - lens.sum()
    off = np.concatenate([[0], np.cumsum(lens)])
    corpus = Corpus(x, off)
    R = a.queries * a.lq
    q = torch.randn((R, a.dim), device="cuda", generator=g)
    q = (q / q.norm(dim=1, keepdim=True)).to(tdt)
    lib = _lib.load()
    s = _lib.CbxBatch()
    s.q_tokens, s.n_q_tokens = q.data_ptr(), R
    s.d_tokens, s.n_d_tokens = x.data_ptr(), a.tokens
    s.dim, s.dtype, s.clamp_negative, s.max_lq = a.dim, dtype_code(tdt), 1, R
    code = {"tc": _lib.CBX_PATH_TC, "simt": _lib.CBX_PATH_SIMT}[a.path]
    wsb = lib.cbx_stage1_workspace_bytes(ctypes.byref(s), a.kp, code)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    tok = torch.empty((R, a.kp), dtype=torch.int64, device="cuda")
    val = torch.empty((R, a.kp), dtype=torch.float64, device="cuda")
    st = torch.zeros(4, dtype=torch.int32, device="cuda")
    norm = corpus.norm_max()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    rb = (R + 127) // 128
    nbytes = a.tokens * a.dim * 2
    print(f"corpus {a.tokens} tokens x {a.dim} ({nbytes / 1e9:.2f} GB), rows {R} ({rb} row blocks), k'={a.kp}, "
          f"path {a.path}, workspace {wsb / 1e6:.1f} MB", flush=True)
    for it in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        _lib.check(lib.cbx_stage1_topk(ctypes.byref(s), a.kp, code, ctypes.c_float(norm), tok.data_ptr(),
                                       val.data_ptr(), st.data_ptr(), ws.data_ptr(), wsb, stream), "stage1")
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        gbs = rb * nbytes / ms / 1e6
        tf = 2.0 * R * a.tokens * a.dim / ms / 1e9
        print(f"iter {it}: {ms:.3f} ms  {gbs:.0f} GB/s (corpus x row blocks)  {tf:.1f} TFLOP/s  status {st.tolist()}",
              flush=True)
    if a.check:
        t0 = time.time()
        ts, vs = stage1_topk(corpus, q, a.kp, True, path="simt")
        print(f"simt check: {time.time() - t0:.2f} s; equal: {np.array_equal(ts, tok.cpu().numpy())} "
              f"{np.array_equal(vs, val.cpu().numpy())}")


if __name__ == "__main__":
    main()
