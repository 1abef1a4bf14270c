"""CPU-side checks of the C ABI: the library loads and exports every declared symbol."""

import ctypes
import os
import re

import pytest

from conftest import ROOT, cuda_available
from paper_2602_02827_b200 import _lib

HEADER = os.path.join(ROOT, "include", "colbandit_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^CBX_API\s+[\w\s\*]+?\b(cbx_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_entry_points():
    syms = declared_symbols()
    for name in ("cbx_maxsim_scores", "cbx_topk_f32", "cbx_rerank_topk", "cbx_maxsim_cells_f64",
                 "cbx_bandit_run", "cbx_last_error", "cbx_abi_version"):
        assert name in syms


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(declared_symbols())
    assert lib.cbx_abi_version() == _lib.CBX_ABI_VERSION == 1


def test_struct_layouts_match_the_header():
    # sizes follow the C layout (natural alignment, 64-bit)
    assert ctypes.sizeof(_lib.CbxBatch) == 5 * 8 + 4 * 8 + 4 * 4 + 2 * 8 + 4 + 4
    assert ctypes.sizeof(_lib.CbxPcg64) == 4 * 8 + 2 * 4
    assert ctypes.sizeof(_lib.CbxBanditOut) == 8 + 4 * 4
    assert ctypes.sizeof(_lib.CbxBanditRunDesc) == 152  # static_assert in csrc/bandit.cu


def test_library_is_sm100a_only():
    path = _lib.LIB_PATH
    data = open(path, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU failure mode")
def test_product_path_fails_loudly_without_a_gpu():
    from paper_2602_02827_b200.batch import TokenBatch

    import numpy as np

    with pytest.raises(RuntimeError, match="CUDA device"):
        TokenBatch.from_host([np.ones((2, 8), np.float16)], [[np.ones((3, 8), np.float16)]])


def test_error_mapping():
    with pytest.raises(ValueError):
        _lib.check(_lib.CBX_EINVAL)
    with pytest.raises(IndexError):
        _lib.check(_lib.CBX_ERANGE)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.CBX_EINTERNAL)


def test_product_package_never_imports_the_test_oracle():
    """The CPU restatement under oracle/ is the checker only: no module of the product may import it
    (``paper_2602_02827_b200.oracle`` is the package's own device-backed MaxSimOracle, imported relatively)."""
    pkg = os.path.join(ROOT, "paper_2602_02827_b200")
    for name in sorted(os.listdir(pkg)):
        if not name.endswith(".py"):
            continue
        src = open(os.path.join(pkg, name)).read()
        assert not re.search(r"^\s*(from\s+oracle\b|import\s+oracle\b)", src, flags=re.M), name


def test_header_constants_match_the_binding():
    """Every numeric ``#define CBX_*`` of the header has the same value in the ctypes binding."""
    src = open(HEADER).read()
    defs = dict(re.findall(r"^#define\s+(CBX_\w+)\s+(-?\d+)\b", src, flags=re.M))
    assert "CBX_BANDIT_MAX_COLS" in defs and "CBX_BANDIT_EDESC" in defs
    missing = [k for k in defs if not hasattr(_lib, k)]
    assert not missing, missing
    for k, v in defs.items():
        assert getattr(_lib, k) == int(v), k


def test_experimental_library_override_needs_the_tools_flag():
    """CBX_LIB alone never redirects the product to another .so (tests, smoke() and bench load the in-tree one)."""
    import subprocess
    import sys

    code = ("import os, sys; sys.path.insert(0, %r); from paper_2602_02827_b200 import _lib; print(_lib.LIB_PATH)"
            % ROOT)
    env = dict(os.environ, CBX_LIB="/tmp/not_the_product.so")
    env.pop("CBX_TOOLS", None)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True).stdout
    assert out.strip() == os.path.join(ROOT, "paper_2602_02827_b200", "libcbx.so")
    env["CBX_TOOLS"] = "1"
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True).stdout
    assert out.strip() == "/tmp/not_the_product.so"
