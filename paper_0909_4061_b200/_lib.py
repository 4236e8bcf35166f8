"""ctypes binding of liblowrank_b200.so (include/lowrank_b200.h).

The library is the product's compute path; there is no CPU fallback.  If
the shared object is missing, or no CUDA device is visible, every call
raises -- loudly -- instead of silently computing elsewhere.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LOWRANK_B200_LIB", os.path.join(_HERE, "liblowrank_b200.so"))

F32, F64, C64, C128 = 0, 1, 2, 3
OP_N, OP_T, OP_C = 0, 1, 2
F32_SPLIT3, F32_SIMT = 0, 1

OK, EINVAL, ECONV, ENOTPSD, ECUDA, ENOMEM, EUNSUPPORTED = range(7)


class LibraryMissing(RuntimeError):
    """liblowrank_b200.so could not be loaded (build it with build())."""


class ConvergenceError(RuntimeError):
    """An iterative kernel failed to converge (reference core.py:25-26)."""


class NotPSDError(ValueError):
    """Cholesky pivot too negative (reference core.py:29-30)."""


_i64 = C.c_int64
_vp = C.c_void_p
_int = C.c_int

# name -> argtypes (all return int except where noted)
_SIGS = {
    "lr_abi_version": [],
    "lr_create": [_int, _vp, C.POINTER(_vp)],
    "lr_destroy": [_vp],
    "lr_set_stream": [_vp, _vp],
    "lr_set_f32_mode": [_vp, _int],
    "lr_reserve": [_vp, _i64],
    "lr_gemm": [_vp, _int, _int, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64],
    "lr_gemm_f64acc": [_vp, _int, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64],
    "lr_gemm_scaled": [_vp, _int, _int, _i64, _i64, _i64, _vp, _i64, C.c_double, _vp, _i64, _vp,
                       _i64],
    "lr_gram": [_vp, _int, _i64, _i64, _vp, _i64, _vp],
    "lr_gram_tc": [_vp, _i64, _i64, _vp, _i64, _vp, _int, _vp],
    "lr_ozaki_prepare": [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp],
    "lr_ozaki_prepare_rows": [_vp, _i64, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp],
    "lr_gemm_ozaki": [_vp, _int, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _i64],
    "lr_chol_drop": [_vp, _int, _i64, _vp, C.c_double, C.c_double, C.c_double, _vp, _vp, _vp],
    "lr_chol_psd": [_vp, _int, _i64, _vp, C.c_double, _vp, _vp, _vp],
    "lr_herm_prep": [_vp, _int, _i64, _vp, _i64, _vp, C.c_double, _int, _vp],
    "lr_eig_finish": [_vp, _int, _i64, _vp, _vp, _vp, _vp, _vp],
    "lr_chol_drop_fast": [_vp, _int, _i64, _vp, C.c_double, C.c_double, C.c_double, C.c_double,
                          _vp, _vp, _vp, _vp],
    "lr_orth": [_vp, _int, _i64, _i64, _vp, _i64, _vp, _i64, C.c_double, C.POINTER(_i64)],
    "lr_small_svd": [_vp, _int, _i64, _i64, _vp, _vp, _vp, _vp],
    "lr_orth_fast": [_vp, _int, _i64, _i64, _vp, _i64, _vp, _i64, C.c_double, _vp],
    "lr_orth_fast_deferred": [_vp, _int, _i64, _i64, _vp, _i64, _vp, _vp, C.c_double, _vp],
    "lr_small_svd_fast": [_vp, _int, _i64, _i64, _vp, _vp, _vp, _vp, _vp],
    "lr_jacobi_svd": [_vp, _int, _i64, _vp, _vp, _vp, _vp, _vp],
    "lr_estimate_tail": [_vp, _int, _i64, _i64, _i64, _vp, _i64, _vp, _i64, C.c_double, _vp],
    "lr_srft": [_vp, _int, _i64, _i64, _i64, _vp, _i64, _vp, _vp, C.c_double, _vp, _i64],
    "lr_srft_scaled": [_vp, _int, _i64, _i64, _i64, _vp, _i64, C.c_double, _vp, _vp, C.c_double,
                       _vp, _i64],
    "lr_dft_rows": [_vp, _int, _i64, _i64, _vp, _i64],
    "lr_gsrft_matrix": [_vp, _int, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                        C.c_double, _vp],
    "lr_csr_spmm": [_vp, _int, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _int],
    "lr_check_finite": [_vp, _int, _i64, _i64, _vp, _i64, _vp, _vp],
    "lr_copy": [_vp, _int, _vp, _i64, _int, _vp, _i64, _i64, _i64, _int],
    "lr_sign_fix": [_vp, _int, _i64, _i64, _i64, _vp, _i64, _vp, _i64],
    "lr_max_abs_imag": [_vp, _int, _i64, _i64, _vp, _i64, _vp],
    "lr_gaussian": [_vp, C.c_uint64, C.c_uint64, _i64, _int, _vp, _vp],
    "lr_axpy_sub": [_vp, _int, _i64, _i64, _vp, _i64, _vp, _i64],
    "lr_axpy_add": [_vp, _int, _i64, _i64, _vp, _i64, _vp, _i64],
    "lr_sylvester_div": [_vp, _int, _i64, _i64, _vp, _i64, _vp, _vp, C.c_double],
    "lr_col_sumsq": [_vp, _int, _i64, _i64, _vp, _i64, _vp],
    "lr_row_id": [_vp, _int, _i64, _i64, _i64, _vp, _i64, _vp, _int, _vp, _i64, _vp],
    "lr_comm_unique_id": [_vp],
    "lr_comm_init": [_vp, _vp, _int, _int],
    "lr_comm_destroy": [_vp],
    "lr_comm_allreduce": [_vp, _int, _i64, _vp],
    "lr_orth_sharded": [_vp, _int, _i64, _i64, _vp, _i64, _vp, _i64, C.c_double, _vp],
    "lr_scale_col": [_vp, _int, _i64, _vp, _i64, C.c_double, _vp, _i64],
}

_lib = None
_lock = threading.Lock()


def exported_symbols():
    return sorted(_SIGS) + ["lr_last_error", "lr_workspace_bytes", "lr_launch_count",
                            "lr_pool_generation"]


# kernels launched through CUDA-graph replays (factor._replay): the C
# counter sees each captured kernel once, at capture time
GRAPH_LAUNCHES = [0]


def launch_count():
    """This library's kernels launched so far: direct launches + graph replays."""
    return int(load().lr_launch_count()) + GRAPH_LAUNCHES[0]


def load():
    """Load the shared library (no GPU needed just to load it)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not found: run `python -m paper_0909_4061_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        lib = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _int
        lib.lr_last_error.argtypes = []
        lib.lr_last_error.restype = C.c_char_p
        lib.lr_workspace_bytes.argtypes = [_vp]
        lib.lr_workspace_bytes.restype = _i64
        lib.lr_launch_count.argtypes = []
        lib.lr_launch_count.restype = C.c_uint64
        lib.lr_pool_generation.argtypes = [_vp]
        lib.lr_pool_generation.restype = C.c_uint64
        _lib = lib
    return _lib


def check(status):
    if status == OK:
        return
    msg = load().lr_last_error().decode(errors="replace")
    if status == EINVAL:
        raise ValueError(msg)
    if status == ECONV:
        raise ConvergenceError(msg)
    if status == ENOTPSD:
        raise NotPSDError(msg)
    if status == EUNSUPPORTED:
        raise NotImplementedError(msg)
    if status == ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"liblowrank_b200: {msg} (status {status})")


HOST_PROFILE = {} if os.environ.get("LR_PROFILE_HOST") else None


def call(name, *args):
    if HOST_PROFILE is None:
        check(getattr(load(), name)(*args))
        return
    import time
    t0 = time.perf_counter()
    check(getattr(load(), name)(*args))
    dt = time.perf_counter() - t0
    c, s = HOST_PROFILE.get(name, (0, 0.0))
    HOST_PROFILE[name] = (c + 1, s + dt)


# ---------------------------------------------------------------------------
# handles: one per (thread, device); the stream is torch's current stream at
# every call, so the library is stream-ordered with the surrounding torch work.

_tls = threading.local()


def handle(device=None):
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_0909_4061_b200 needs a CUDA device (no CPU fallback)")
    dev = torch.cuda.current_device() if device is None else int(device)
    hs = getattr(_tls, "handles", None)
    if hs is None:
        hs = _tls.handles = {}
    h = hs.get(dev)
    lib = load()
    stream = torch.cuda.current_stream(dev).cuda_stream
    if h is None:
        hp = _vp()
        with torch.cuda.device(dev):
            check(lib.lr_create(dev, _vp(stream), C.byref(hp)))
        h = hs[dev] = hp
    else:
        check(lib.lr_set_stream(h, _vp(stream)))
    return h


def pool_generation(h):
    """Generation of handle h's scratch pool (lr_pool_generation)."""
    return int(load().lr_pool_generation(h))


def set_f32_mode(mode, device=None):
    call("lr_set_f32_mode", handle(device), int(mode))


# ---------------------------------------------------------------------------
# dtype helpers

def dtype_code(t):
    import torch
    m = {torch.float32: F32, torch.float64: F64, torch.complex64: C64, torch.complex128: C128}
    if t not in m:
        raise ValueError(f"unsupported dtype {t}")
    return m[t]


def wide_torch(code):
    import torch
    return torch.complex128 if code in (C64, C128) else torch.float64


def ptr(t):
    return _vp(t.data_ptr()) if t is not None else _vp(0)


def ld(t):
    """Row stride of a 2-D row-major tensor (unit column stride required)."""
    if t.dim() == 1:
        return 1
    if t.shape[1] > 1 and t.stride(1) != 1:
        raise ValueError("expected a row-major (unit column stride) tensor")
    if t.shape[0] <= 1:
        return max(1, int(t.shape[1]))
    return int(t.stride(0))


def np_dtype(code):
    return {F32: np.float32, F64: np.float64, C64: np.complex64, C128: np.complex128}[code]
