"""ctypes binding of libcbx.so (the C ABI in include/colbandit_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (plain
``nvcc -shared``, sm_100a). There is no fallback: if the library or a CUDA
device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcbx.so")
# A/B tooling only (tools/p2var.sh, tools/ab_packed.py): CBX_LIB names an experimental build, and it is honoured
# only together with CBX_TOOLS=1 so that no test, smoke() or bench run can load anything but the in-tree library.
if os.environ.get("CBX_TOOLS") == "1" and os.environ.get("CBX_LIB"):
    LIB_PATH = os.environ["CBX_LIB"]

CBX_ABI_VERSION = 1
CBX_OK, CBX_EINVAL, CBX_ERANGE, CBX_ECUDA, CBX_EINTERNAL = 0, 1, 2, 3, 4
CBX_F32, CBX_F16, CBX_BF16, CBX_F64 = 0, 1, 2, 3
CBX_PATH_AUTO, CBX_PATH_TC, CBX_PATH_SIMT = 0, 1, 2
CBX_EPSILON_GREEDY, CBX_STATIC_WARMUP, CBX_UNIFORM_ROW = 0, 1, 2
CBX_TERM_SEPARATION, CBX_TERM_EXHAUSTION = 0, 1
CBX_BANDIT_ROW_SLACK = 64
CBX_BANDIT_TREE = 1
CBX_BANDIT_PREWARMED = 2
CBX_BANDIT_MAX_COLS = 128
CBX_BANDIT_EDESC = 3
CBX_BANDIT_STEP_BYTES = 256
CBX_SHARD_REVEAL, CBX_SHARD_WARMUP, CBX_SHARD_DONE = 0, 1, 2
CBX_IPC_HANDLE_BYTES = 64


class CbxMboxPeer(ctypes.Structure):
    _fields_ = [("val", ctypes.c_void_p), ("flag", ctypes.c_void_p)]


class CbxBatch(ctypes.Structure):
    _fields_ = [
        ("q_tokens", ctypes.c_void_p),
        ("q_tok_off", ctypes.c_void_p),
        ("d_tokens", ctypes.c_void_p),
        ("d_tok_off", ctypes.c_void_p),
        ("q_doc_off", ctypes.c_void_p),
        ("n_queries", ctypes.c_int64),
        ("n_docs", ctypes.c_int64),
        ("n_q_tokens", ctypes.c_int64),
        ("n_d_tokens", ctypes.c_int64),
        ("dim", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("clamp_negative", ctypes.c_int32),
        ("max_lq", ctypes.c_int32),
        ("max_q_docs", ctypes.c_int64),
        ("max_q_doc_tokens", ctypes.c_int64),
        ("d_norm_max", ctypes.c_float),
        ("reserved", ctypes.c_int32),
    ]


class CbxPcg64(ctypes.Structure):
    _fields_ = [
        ("state_hi", ctypes.c_uint64),
        ("state_lo", ctypes.c_uint64),
        ("inc_hi", ctypes.c_uint64),
        ("inc_lo", ctypes.c_uint64),
        ("has_uint32", ctypes.c_uint32),
        ("uinteger", ctypes.c_uint32),
    ]


class CbxBanditRunDesc(ctypes.Structure):
    _fields_ = [
        ("query", ctypes.c_int64),
        ("row_begin", ctypes.c_int64),
        ("n_rows", ctypes.c_int32),
        ("n_cols", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("explore_mode", ctypes.c_int32),
        ("n_warm", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("warm_off", ctypes.c_int64),
        ("alpha_ef", ctypes.c_double),
        ("epsilon", ctypes.c_double),
        ("log_term", ctypes.c_double),
        ("bounds_off", ctypes.c_int64),
        ("lo_uniform", ctypes.c_double),
        ("hi_uniform", ctypes.c_double),
        ("trace_off", ctypes.c_int64),
        ("state_off", ctypes.c_int64),
        ("rng", CbxPcg64),
    ]


class CbxBanditOut(ctypes.Structure):
    _fields_ = [
        ("n_reveals", ctypes.c_int64),
        ("iterations", ctypes.c_int32),
        ("terminated_by", ctypes.c_int32),
        ("status", ctypes.c_int32),
        ("pad", ctypes.c_int32),
    ]


# every symbol include/colbandit_b200.h declares, with its ctypes signature
_P = ctypes.c_void_p
_I = ctypes.c_int
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_SZ = ctypes.c_size_t
SIGNATURES = {
    "cbx_abi_version": (_I, []),
    "cbx_last_error": (ctypes.c_char_p, []),
    "cbx_device_info": (_I, [_P, _P, _P]),
    "cbx_workspace_bytes": (_SZ, [_P, _I]),
    "cbx_maxsim_scores": (_I, [_P, _P, _I, _P, _SZ, _P]),
    "cbx_topk_f32": (_I, [_P, _P, _I64, _I64, _I, _P, _P, _P, _SZ, _P]),
    "cbx_topk_f64": (_I, [_P, _P, _I64, _I64, _I, _P, _P, _P, _SZ, _P]),
    "cbx_rerank_topk": (_I, [_P, _I, _I, _P, _P, _P, _P, _SZ, _P]),
    "cbx_maxsim_cells_f64": (_I, [_P, _P, _I64, _P, _P]),
    "cbx_corpus_workspace_bytes": (_SZ, [_I64, _I64, _I64, _I]),
    "cbx_corpus_rerank_topk": (_I, [_P, _P, _I64, _P, _I, _P, _P, _P, _P, _P, _SZ, _P]),
    "cbx_gather_candidates": (_I, [_P, _P, _I64, _I, _I, _P, _I64, _P, _I64, _P, _P, _P]),
    "cbx_row_partial_fsum": (_I, [_P, _I64, _P, _I64, _I, _P, _P, _P]),
    "cbx_stage1_workspace_bytes": (_SZ, [_P, _I, _I]),
    "cbx_stage1_topk": (_I, [_P, _I, _I, ctypes.c_float, _P, _P, _P, _P, _SZ, _P]),
    "cbx_token_norm_max": (_I, [_P, _I64, _I, _I, _P, _P]),
    "cbx_bandit_state_bytes": (_SZ, [_I64]),
    "cbx_bandit_set_profile": (None, [_P]),
    "cbx_bandit_set_row_cache": (None, [_P, _P]),
    "cbx_bandit_set_row_cache_threshold": (None, [ctypes.c_int]),
    "cbx_pcg64_draws": (_I, [_P, _P, _I64, _P, _P, _P]),
    "cbx_bandit_shard_run": (_I, [_P, _P, _I64, _P, _I32, _P, _I32, _I32, _P, _I32, _P, _P, _P, _P, _SZ, _P, _I32, _P,
                                  _P, _P, _P, _P]),
    "cbx_mbox_alloc": (_I, [_I64, _P, _P]),
    "cbx_mbox_free": (_I, [_P]),
    "cbx_mbox_clear": (_I, [_P, _I64, _P]),
    "cbx_mbox_view": (_I, [_P, _I64, _P]),
    "cbx_ipc_get_handle": (_I, [_P, _P]),
    "cbx_ipc_open": (_I, [_P, _P]),
    "cbx_ipc_close": (_I, [_P]),
    "cbx_bandit_run": (_I, [_P, _P, _I64, _P, _I64, _I32, _P, _P, _P, _P, _SZ, _P, _I32, _P, _P, _P, _P, _P]),
    "cbx_bandit_prewarm": (_I, [_P, _P, _I64, _P, _I64, _P, _P, _P, _P, _P]),
    "cbx_bandit_shard_step": (_I, [_P, _P, _I64, _P, _I64, _I64, _I, _P, _P, _P, _P, _SZ, _P, _P, _P, _I32, _P, _P,
                                   _P, _P, _P]),
}

_lib = None
_lock = threading.Lock()


class CbxError(RuntimeError):
    pass


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libcbx.so once; raise loudly if it was not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise ImportError(
                    f"{path} is missing: build the CUDA extension with `python -c 'import __graft_entry__ as g; g.build()'`"
                )
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().cbx_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == CBX_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == CBX_EINVAL:
        raise ValueError(msg)
    if rc == CBX_ERANGE:
        raise IndexError(msg)
    raise CbxError(msg)


def require_cuda():
    """The product path runs on the GPU only; there is no CPU fallback."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2602_02827_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    load()
    return torch
