"""The C-ABI library loads without a GPU and exports every entry point that
include/lowrank_b200.h declares (no compute calls here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lowrank_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lr_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_boundary():
    names = declared()
    for must in ("lr_create", "lr_gemm", "lr_orth", "lr_small_svd", "lr_srft", "lr_csr_spmm",
                 "lr_estimate_tail", "lr_gram", "lr_chol_drop"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_0909_4061_b200 import _lib
    lib = _lib.load()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, f"not exported: {missing}"
    assert lib.lr_abi_version() == 1
    # the Python binding covers every declared entry point
    assert set(declared()) <= set(_lib.exported_symbols())


def test_library_is_sm100a():
    from paper_0909_4061_b200 import _lib
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_product_path_has_no_oracle_import():
    """The product package never imports the CPU oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_0909_4061_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), fn
            assert "lowrank_oracle" not in src, fn
