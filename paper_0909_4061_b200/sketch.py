"""Random test matrices and the SRFT fast apply.

Mirrors the hot-path part of the reference's ``lowrank.sketch``
(/root/reference/pkg/src/lowrank/sketch.py).  Random draws follow the
reference's counter-based Philox keying (sketch.py:32-42) so the same
(dimensions, seed) give bitwise the same Omega / D / R as the reference:
Gaussian matrices are drawn on the device (lr_gaussian), the SRFT's D and R on
the host (the permutation is sequential) and uploaded.  The SRFT runs as the
shared-memory FFT (power-of-two n) or as a pass over A against the picked,
D-scaled DFT columns (any n -- the linear map the reference evaluates with
Bluestein for non-power-of-two lengths, sketch.py:155-176).  The
Givens-chain variant (GSRFT) builds the ell picked columns of its Omega on
the device (two rotation chains, permutations and diagonals applied to the
picked DFT columns) and is then one pass over A as well.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import _out, _torch, is_device_array, to_device

_STREAM_GAUSS = 0x67617573
_STREAM_SRFT = 0x73726674
_STREAM_GSRFT = 0x67737266
_STREAM_ORTHO = 0x6F727468


def rng_for(seed, stream=0, index=0):
    """Philox generator keyed by seed | stream<<64 | index<<96 (sketch.py:32-42)."""
    key = (int(seed) & (2**64 - 1)) | ((int(stream) & (2**32 - 1)) << 64) | (
        (int(index) & (2**32 - 1)) << 96)
    return np.random.Generator(np.random.Philox(key=key))


# ---------------------------------------------------------------------------
# operation counter (reference sketch.py:45-62): one process-wide counter of
# the scalar operations the structured-sketch applications perform, in the
# reference's cost units (complex multiply 6, complex add 2).  The counts are
# those of the path that actually ran on the device: the FFT kernels (radix-16
# Stockham for power-of-two n) are charged the reference's own radix-2 model
# (D: 6 n, butterflies 10 n/2 per level, normalization 2 n, picks 2 ell per
# row -- an upper bound of the radix-16 work), the dense picked-DFT-column
# product (non-power-of-two n, LR_SRFT=gemm, the GSRFT's picked columns)
# 8 n ell per row.

_OPS = 0


def reset_op_count():
    global _OPS
    _OPS = 0


def op_count():
    return _OPS


def _count(n):
    global _OPS
    _OPS += int(n)


def _fft_model_ops(rows, n):
    """Reference cost of one unitary length-n DFT per row (sketch.py:146,199)."""
    lg = int(n).bit_length() - 1
    return 10 * rows * (n // 2) * lg + 2 * rows * n


def _srft_uses_fft(n, dtype):
    """Whether srft.cu runs an FFT kernel for this length (else the dense
    picked-column product)."""
    import os
    torch = _torch()
    mode = os.environ.get("LR_SRFT", "")
    es = 8 if dtype in (torch.complex64, torch.float32) else 16
    return (n >= 1 and (n & (n - 1)) == 0 and not mode.startswith("g")
            and n * es <= 200 * 1024)


@dataclass
class SketchSpec:
    """Configuration of one randomized sketch draw (sketch.py:69-93)."""

    kind: str = "gaussian"
    ell: int = 1
    power_q: int = 0
    seed: int = 0

    def __post_init__(self):
        if self.kind not in ("gaussian", "srft", "gsrft"):
            raise ValueError(f"unknown sketch kind {self.kind!r}")
        if self.ell < 1:
            raise ValueError("sample count ell must be >= 1")
        if self.power_q < 0:
            raise ValueError("power exponent must be nonnegative")

    @classmethod
    def fixed_rank(cls, kind, k, p=5, q=0, seed=0):
        return cls(kind=kind, ell=int(k) + int(p), power_q=q, seed=seed)


def gaussian_matrix(n, ell, seed):
    """n-by-ell i.i.d. standard normals keyed by seed (sketch.py:96-100).

    This is the reference-API function: a numpy array drawn on the host
    (bitwise identical to the reference).  The range finders do not call it:
    they draw the same stream on the device (gaussian_dev)."""
    if n < 1 or ell < 1:
        raise ValueError("dimensions must be >= 1")
    return rng_for(seed, _STREAM_GAUSS).standard_normal((n, ell))


def gaussian_dev(n, ell, seed, stream=_STREAM_GAUSS, index=0, dtype=None, device=None):
    """The same n x ell draw as gaussian_matrix / rng_for(seed, stream,
    index).standard_normal((n, ell)), generated on the GPU (K0 kernel: the
    Philox4x64-10 stream and numpy's ziggurat).  Returns a CUDA tensor in
    `dtype` (float64 default; float32 is numpy's astype rounding)."""
    torch = _torch()
    from .core import _SPEC
    dt = torch.float64 if dtype is None else dtype
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    out = torch.empty((n, ell), dtype=dt, device=dev)
    key_lo = int(seed) & (2**64 - 1)
    key_hi = (int(stream) & (2**32 - 1)) | ((int(index) & (2**32 - 1)) << 32)
    st = _SPEC.status
    local = st is None
    if local:
        st = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("lr_gaussian", _lib.handle(dev.index), key_lo, key_hi, n * ell,
              _lib.dtype_code(dt), _lib.ptr(out), _lib.ptr(st))
    if local and int(st.item()) != 0:
        raise RuntimeError("device Gaussian stream: ziggurat cap exceeded (status %d)" % int(st.item()))
    return out


@dataclass
class SrftOperator:
    """Materialized SRFT draw: scale * D F R with unimodular diagonal d
    (sketch.py:207-218)."""

    n: int
    ell: int
    d: np.ndarray
    picks: np.ndarray
    scale: float

    def to_dense(self):
        return srft_apply(np.eye(self.n), self)


def srft_operator(n, ell, seed):
    """d = exp(2 pi i U[0,1)) then picks = permutation(n)[:ell], one stream
    (sketch.py:250-256)."""
    if ell > n:
        raise ValueError("sample count exceeds dimension")
    rng = rng_for(seed, _STREAM_SRFT)
    d = np.exp(2j * np.pi * rng.random(n))
    picks = rng.permutation(n)[:ell]
    return SrftOperator(n=n, ell=ell, d=d, picks=picks, scale=float(np.sqrt(n / ell)))


def _resolve(spec_or_op, n, op_type=None, builder=None):
    """Materialize a SketchSpec (or pass an operator through), as the
    reference's _resolve (sketch.py:294-303)."""
    op_type = op_type or SrftOperator
    builder = builder or srft_operator
    if isinstance(spec_or_op, op_type):
        op = spec_or_op
    elif isinstance(spec_or_op, SketchSpec):
        op = builder(n, spec_or_op.ell, spec_or_op.seed)
    else:
        raise TypeError("expected a SketchSpec or a materialized operator")
    if op.n != n:
        raise ValueError("operator dimension does not match matrix columns")
    return op


def _complex_of(t):
    """Complex compute dtype for an input tensor (real inputs are promoted,
    as in the reference's A * d, sketch.py:315)."""
    torch = _torch()
    if t.dtype in (torch.complex64, torch.float32):
        return torch.complex64
    return torch.complex128


def _device_cached(op, key, make):
    """Device copies derived from a (host-drawn) sketch operator, kept on the
    operator object: a repeated randomized SVD with the same draw uploads
    nothing, so its step has no host->device copy (which would synchronize
    the stream) and can be captured as a CUDA graph."""
    cache = op.__dict__.setdefault("_dev_cache", {})
    val = cache.get(key)
    if val is None:
        val = cache[key] = make()
    return val


_OPERATORS = {}


def cached_operator(kind, n, ell, seed):
    """srft_operator / gsrft_operator(n, ell, seed), memoized (the draws are
    a pure function of the arguments; bounded cache)."""
    key = (kind, int(n), int(ell), int(seed))
    op = _OPERATORS.get(key)
    if op is None:
        op = (srft_operator if kind == "srft" else gsrft_operator)(n, ell, seed)
        if len(_OPERATORS) >= 16:
            _OPERATORS.pop(next(iter(_OPERATORS)))
        _OPERATORS[key] = op
    return op


def srft_dev(A, op, amax=None):
    """Y = scale * dft(A o d)[:, picks] for a device matrix A (K5).  amax:
    max |A| when known (DenseOperator.amax) -- complex64 runs as one
    tensor-core pass over A (lr_srft_scaled)."""
    torch = _torch()
    m, n = A.shape
    cdt = _complex_of(A)
    code = _lib.dtype_code(cdt)
    h = _lib.handle(A.device.index)
    if A.dtype != cdt:
        Ac = torch.empty((m, n), dtype=cdt, device=A.device)
        _lib.call("lr_copy", h, _lib.dtype_code(A.dtype), _lib.ptr(A), _lib.ld(A), code,
                  _lib.ptr(Ac), _lib.ld(Ac), m, n, 0)
        A = Ac
    d, picks = _device_cached(op, ("srft", cdt, A.device.index), lambda: (
        torch.from_numpy(np.ascontiguousarray(op.d)).to(device=A.device, dtype=cdt),
        torch.from_numpy(np.ascontiguousarray(op.picks, dtype=np.int32)).to(A.device)))
    Y = torch.empty((m, op.ell), dtype=cdt, device=A.device)
    _lib.call("lr_srft_scaled", h, code, m, n, op.ell, _lib.ptr(A), _lib.ld(A),
              float(-1.0 if amax is None else amax), _lib.ptr(d), _lib.ptr(picks),
              float(op.scale), _lib.ptr(Y), _lib.ld(Y))
    _count_srft(m, n, op.ell, cdt)
    return Y


def _count_srft(rows, n, ell, dtype):
    if _srft_uses_fft(n, dtype):
        _count(6 * rows * n + _fft_model_ops(rows, n) + 2 * rows * ell)
    else:
        _count(8 * rows * n * ell + 2 * rows * ell)


def srft_apply(A, spec_or_op):
    """Y = A @ Omega for an SRFT Omega (sketch.py:306-320), on the GPU.

    The result is complex and agrees with the explicit dense product to
    roundoff of the compute precision."""
    host = not is_device_array(A)
    t = to_device(A)
    if t.dim() != 2:
        raise ValueError("A must be 2-D")
    op = _resolve(spec_or_op, t.shape[1])
    return _out(srft_dev(t, op), host)


def dft(v, axis=-1):
    """Unitary DFT along `axis`, f_pq = n^-1/2 exp(-2 pi i pq / n)
    (sketch.py:179-200), any length."""
    torch = _torch()
    host = not is_device_array(v)
    t = to_device(v)
    if t.dim() == 0:
        raise ValueError("dft expects a vector or matrix")
    t = torch.movedim(t, axis, -1)
    shape = t.shape
    n = shape[-1]
    cdt = _complex_of(t)
    X = t.to(cdt).reshape(-1, n).contiguous()
    if n > 1:
        # power of two: shared-memory radix-16 FFT; otherwise the dense DFT
        # matrix product (same linear map as the reference's Bluestein path)
        _lib.call("lr_dft_rows", _lib.handle(X.device.index), _lib.dtype_code(cdt), X.shape[0], n,
                  _lib.ptr(X), _lib.ld(X))
        _count(_fft_model_ops(X.shape[0], n) if (n & (n - 1)) == 0 else 8 * X.shape[0] * n * n)
    out = torch.movedim(X.reshape(shape), -1, axis)
    return _out(out, host)


@dataclass
class GsrftOperator:
    """Givens-chain SRFT draw (sketch.py:221-243): applied to a row vector x
    as x D'' Theta' D' Theta D F R, each Theta a random permutation followed
    by the ascending chain of plane rotations G(i, i+1; theta_i)."""

    n: int
    ell: int
    d_outer: np.ndarray
    perm_outer: np.ndarray
    thetas_outer: np.ndarray
    d_mid: np.ndarray
    perm_inner: np.ndarray
    thetas_inner: np.ndarray
    d_inner: np.ndarray
    picks: np.ndarray
    scale: float

    def to_dense(self):
        return gsrft_apply(np.eye(self.n), self)


def gsrft_operator(n, ell, seed):
    """Draw order of sketch.py:259-275 (one Philox stream, host side)."""
    if ell > n:
        raise ValueError("sample count exceeds dimension")
    rng = rng_for(seed, _STREAM_GSRFT)

    def unimodular():
        return np.exp(2j * np.pi * rng.random(n))

    d_outer = unimodular()
    perm_outer = rng.permutation(n)
    thetas_outer = rng.uniform(0.0, 2.0 * np.pi, max(n - 1, 0))
    d_mid = unimodular()
    perm_inner = rng.permutation(n)
    thetas_inner = rng.uniform(0.0, 2.0 * np.pi, max(n - 1, 0))
    d_inner = unimodular()
    picks = rng.permutation(n)[:ell]
    return GsrftOperator(n=n, ell=ell, d_outer=d_outer, perm_outer=perm_outer,
                         thetas_outer=thetas_outer, d_mid=d_mid, perm_inner=perm_inner,
                         thetas_inner=thetas_inner, d_inner=d_inner, picks=picks,
                         scale=float(np.sqrt(n / ell)))


def gsrft_matrix_dev(op, dtype, device):
    """The ell picked columns of the GSRFT (n x ell, complex) built on the
    device (lr_gsrft_matrix): gsrft_apply(A) = A @ this."""
    torch = _torch()
    dev = torch.device("cuda", device)

    def c(x):
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).to(dev)

    def i32(x):
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.int32)).to(dev)

    def f64(x):
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)

    arrs = (c(op.d_outer), i32(op.perm_outer), f64(op.thetas_outer), c(op.d_mid),
            i32(op.perm_inner), f64(op.thetas_inner), c(op.d_inner), i32(op.picks))
    X = torch.empty((op.n, op.ell), dtype=dtype, device=dev)
    _lib.call("lr_gsrft_matrix", _lib.handle(device), _lib.dtype_code(dtype), op.n, op.ell,
              *[_lib.ptr(a) for a in arrs], float(op.scale), _lib.ptr(X))
    return X


def gsrft_dev(A, op, amax=None):
    """Y = A Omega_gsrft for a device matrix A: the picked columns of Omega
    are built on the device, then one pass over A (lr_gemm_scaled)."""
    from .core import _pass
    torch = _torch()
    m, n = A.shape
    cdt = _complex_of(A)
    if A.dtype != cdt:
        Ac = torch.empty((m, n), dtype=cdt, device=A.device)
        _lib.call("lr_copy", _lib.handle(A.device.index), _lib.dtype_code(A.dtype), _lib.ptr(A),
                  _lib.ld(A), _lib.dtype_code(cdt), _lib.ptr(Ac), _lib.ld(Ac), m, n, 0)
        A = Ac
    X = _device_cached(op, ("gsrft", cdt, A.device.index),
                       lambda: gsrft_matrix_dev(op, cdt, A.device.index))
    Y = torch.empty((m, op.ell), dtype=cdt, device=A.device)
    _pass(A, X, Y, False, amax)
    _count(8 * m * n * op.ell + 2 * m * op.ell)
    return Y


def gsrft_apply(A, spec_or_op):
    """Y = A @ Omega for a Givens-chain SRFT Omega (sketch.py:323-337), on the
    GPU; same contract as srft_apply."""
    host = not is_device_array(A)
    t = to_device(A)
    if t.dim() != 2:
        raise ValueError("A must be 2-D")
    op = _resolve(spec_or_op, t.shape[1], GsrftOperator, gsrft_operator)
    return _out(gsrft_dev(t, op), host)


def sketch_apply(A, spec):
    """A @ Omega for the sketch family named in `spec` (sketch.py:340-349):
    Gaussian as one device pass, SRFT / GSRFT through their kernels."""
    host = not is_device_array(A)
    t = to_device(A)
    n = t.shape[1]
    if spec.kind == "gaussian":
        from .core import _cast_like_dtype, gemm
        torch = _torch()
        Om = _cast_like_dtype(gaussian_dev(n, spec.ell, spec.seed, device=t.device.index), t.dtype)
        Y = torch.empty((t.shape[0], spec.ell), dtype=t.dtype, device=t.device)
        gemm(t, Om, Y)
        return _out(Y, host)
    if spec.kind == "srft":
        return srft_apply(A, spec)
    return gsrft_apply(A, spec)


def dense_sketch_matrix(n, spec):
    """The test matrix Omega itself (sketch.py:352-358; the reference's path
    for oracles): Gaussian draws, or the SRFT / GSRFT applied to I_n."""
    if spec.kind == "gaussian":
        return gaussian_matrix(n, spec.ell, spec.seed)
    if spec.kind == "srft":
        return srft_operator(n, spec.ell, spec.seed).to_dense()
    return gsrft_operator(n, spec.ell, spec.seed).to_dense()
