"""Stage A on the GPU: randomized construction of an orthonormal range basis.

Mirrors the fixed-rank range finders of the reference's
``lowrank.rangefinder`` (/root/reference/pkg/src/lowrank/rangefinder.py)
with identical signatures, validation, pass counting and RangeBasis fields.
The sketch Omega and the estimator probes are drawn on the host with the
reference's Philox streams (bitwise identical) and uploaded; the passes over
A, the orthonormalizations and the estimator tail run on the device and the
sample / basis panels stay in HBM between steps.  The adaptive
(fixed-precision) finder is outside this build's scope.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib, config
from .core import (MatVecOperator, _out, _torch, apply_dev, as_operator, cast_dev,
                   is_device_array, orth_dev, to_device)
from .sketch import SketchSpec, gaussian_dev, srft_dev, srft_operator

_STREAM_PROBE = 0x70726F62


@dataclass
class RangeBasis:
    """Orthonormal basis with draw provenance (rangefinder.py:35-46)."""

    Q: object
    samples_used: int
    passes: int
    est_error: float | None
    spec: SketchSpec
    saturated: bool = False
    probe_matvecs: int = 0
    diagnostics: dict = field(default_factory=dict)


def _host_io(A, op):
    """numpy in -> numpy out; device tensors / device operators -> torch."""
    if isinstance(A, MatVecOperator) or hasattr(A, "apply"):
        return getattr(op, "host_io", not op.device_native)
    return not is_device_array(A)


def _op_dtype(op):
    torch = _torch()
    if getattr(op, "device_native", False) and hasattr(op, "dtype"):
        return op.dtype
    return torch.float64


def _real_of(dt):
    torch = _torch()
    return torch.float32 if dt in (torch.float32, torch.complex64) else torch.float64


def _sketch_dev(op, ell, seed):
    """Omega = gaussian_matrix(n, ell, seed) (sketch.py:96-100), drawn on the
    device from the same Philox stream, in the operator's real precision."""
    return gaussian_dev(op.n, ell, seed, dtype=_real_of(_op_dtype(op)))


def _check_ell(op, ell):
    if not 1 <= ell <= min(op.shape):
        raise ValueError("ell must satisfy 1 <= ell <= min(m, n)")


def _cast_like_op(op, X):
    """Real sketches are applied to complex operators as complex arrays."""
    return cast_dev(X, _op_dtype(op))


def randomized_range_finder(A, ell, seed, ortho_tol=config.GS_DROP_TOL):
    """Alg 4.1 (rangefinder.py:49-62): Q = orth(A Omega), one pass.

    A zero sample matrix yields a zero-column basis with est_error 0."""
    op = as_operator(A)
    _check_ell(op, ell)
    spec = SketchSpec(kind="gaussian", ell=ell, seed=seed)
    Y = apply_dev(op, _cast_like_op(op, _sketch_dev(op, ell, seed)))
    Q = orth_dev(Y, ortho_tol)
    est = 0.0 if Q.shape[1] == 0 else None
    return RangeBasis(Q=_out(Q, _host_io(A, op)), samples_used=ell, passes=1, est_error=est,
                      spec=spec)


def _plain_gs_dev(Y):
    """Single-pass Gram-Schmidt with no reorthogonalization or drops
    (rangefinder.py:169-184: each column is reduced against the already
    normalized ones in order, then normalized if nonzero)."""
    torch = _torch()
    Q = Y.clone()
    m, ell = Q.shape
    code = _lib.dtype_code(Q.dtype)
    h = _lib.handle(Q.device.index)
    c = torch.empty((1, 1), dtype=Q.dtype, device=Q.device)
    t = torch.empty((m, 1), dtype=Q.dtype, device=Q.device)
    nrm = torch.empty(1, dtype=torch.float64, device=Q.device)
    ldq = _lib.ld(Q)
    es = Q.element_size()
    base = Q.data_ptr()
    opc = _lib.OP_C if Q.is_complex() else _lib.OP_T
    for j in range(ell):
        qj = _lib._vp(base + j * es)
        for i in range(j):
            qi = _lib._vp(base + i * es)
            # c = q_i^H q_j ; q_j -= q_i c
            _lib.call("lr_gemm", h, code, opc, m, 1, 1, qi, ldq, qj, ldq, _lib.ptr(c), 1)
            _lib.call("lr_gemm", h, code, _lib.OP_N, m, 1, 1, qi, ldq, _lib.ptr(c), 1,
                      _lib.ptr(t), 1)
            _lib.call("lr_axpy_sub", h, code, m, 1, _lib.ptr(t), 1, qj, ldq)
        _lib.call("lr_col_sumsq", h, code, m, 1, qj, ldq, _lib.ptr(nrm))
        nv = math.sqrt(float(nrm.item()))
        if nv > 0:
            _lib.call("lr_scale_col", h, code, m, qj, ldq, 1.0 / nv, qj, ldq)
    return Q


def power_iteration_range(A, ell, q, seed, ortho_tol=config.GS_DROP_TOL, safeguarded=True):
    """Alg 4.3 (rangefinder.py:187-218): orthonormalize (A A*)^q A Omega.

    q = 0 reproduces the basic finder draw for draw; safeguarded=False uses
    the unsafeguarded single-pass Gram-Schmidt."""
    if q < 0:
        raise ValueError("q must be nonnegative")
    op = as_operator(A)
    _check_ell(op, ell)
    spec = SketchSpec(kind="gaussian", ell=ell, power_q=q, seed=seed)
    Y = apply_dev(op, _cast_like_op(op, _sketch_dev(op, ell, seed)))
    for _ in range(q):
        Y = apply_dev(op, apply_dev(op, Y, adjoint=True))
    Q = orth_dev(Y, ortho_tol) if safeguarded else _plain_gs_dev(Y)
    est = 0.0 if Q.shape[1] == 0 else None
    return RangeBasis(Q=_out(Q, _host_io(A, op)), samples_used=ell, passes=2 * q + 2,
                      est_error=est, spec=spec)


def subspace_iteration_range_dev(op, ell, q, seed, ortho_tol=config.GS_DROP_TOL, omega=None):
    """Alg 4.4 on a device operator; returns the device basis."""
    if omega is None:
        omega = _cast_like_op(op, _sketch_dev(op, ell, seed))
    Q = orth_dev(apply_dev(op, omega), ortho_tol)
    for _ in range(q):
        Qt = orth_dev(apply_dev(op, Q, adjoint=True), ortho_tol)
        Q = orth_dev(apply_dev(op, Qt), ortho_tol)
    return Q


def subspace_iteration_range(A, ell, q, seed, ortho_tol=config.GS_DROP_TOL):
    """Alg 4.4 (rangefinder.py:221-243): re-orthonormalize after every
    application of A and A*; passes = 2q + 2."""
    if q < 0:
        raise ValueError("q must be nonnegative")
    op = as_operator(A)
    _check_ell(op, ell)
    spec = SketchSpec(kind="gaussian", ell=ell, power_q=q, seed=seed)
    Q = subspace_iteration_range_dev(op, ell, q, seed, ortho_tol)
    est = 0.0 if Q.shape[1] == 0 else None
    return RangeBasis(Q=_out(Q, _host_io(A, op)), samples_used=ell, passes=2 * q + 2,
                      est_error=est, spec=spec)


def fast_range_finder(A, ell, seed, kind="srft", ortho_tol=config.GS_DROP_TOL):
    """Alg 4.5 (rangefinder.py:246-266): SRFT sketch + orthonormalization.

    Real inputs are promoted to complex; diagnostics["max_imag_sample"]
    records max |Im Y| for real inputs."""
    torch = _torch()
    if kind not in ("srft", "gsrft"):
        raise ValueError("kind must be 'srft' or 'gsrft'")
    if kind == "gsrft":
        raise NotImplementedError("GSRFT is outside this build's scope (SURVEY.md §8f #3)")
    if isinstance(A, MatVecOperator):
        if not hasattr(A, "array"):
            raise TypeError("fast_range_finder needs a dense matrix")
        host, t, amax = A.host_io, A.array, getattr(A, "amax", None)
    else:
        host = not is_device_array(A)
        t = to_device(A)
        amax = None
    spec = SketchSpec(kind=kind, ell=ell, seed=seed)
    op = srft_operator(t.shape[1], ell, seed)
    Y = srft_dev(t, op, amax=amax)
    diagnostics = {}
    if not t.is_complex():
        out = torch.empty(1, dtype=torch.float64, device=Y.device)
        _lib.call("lr_max_abs_imag", _lib.handle(Y.device.index), _lib.dtype_code(Y.dtype),
                  Y.shape[0], Y.shape[1], _lib.ptr(Y), _lib.ld(Y), _lib.ptr(out))
        diagnostics["max_imag_sample"] = float(out.item())
    Q = orth_dev(Y, ortho_tol)
    est = 0.0 if Q.shape[1] == 0 else None
    return RangeBasis(Q=_out(Q, host), samples_used=ell, passes=1, est_error=est, spec=spec,
                      diagnostics=diagnostics)


def probes_dev(op, r, seed):
    """Estimator probes W (rangefinder.py:78), drawn on the host and uploaded."""
    Wd = gaussian_dev(op.n, r, seed, stream=_STREAM_PROBE, dtype=_real_of(_op_dtype(op)))
    return _cast_like_op(op, Wd)


def posterior_error_estimate_dev(op, Q, r=config.DEFAULT_PROBES, alpha=config.DEFAULT_ALPHA,
                                 seed=0, W=None):
    """Device estimator; returns a 1-element float64 device tensor."""
    torch = _torch()
    if W is None:
        W = probes_dev(op, r, seed)
    Z = apply_dev(op, W)
    Z = Z.contiguous() if Z.stride(-1) != 1 else Z
    est = torch.empty(1, dtype=torch.float64, device=Z.device)
    Qd = cast_dev(Q if is_device_array(Q) else to_device(Q), Z.dtype)
    k = Qd.shape[1] if Qd.dim() == 2 else 0
    _lib.call("lr_estimate_tail", _lib.handle(Z.device.index), _lib.dtype_code(Z.dtype),
              Z.shape[0], k, r, _lib.ptr(Qd) if k else _lib.ptr(None), _lib.ld(Qd) if k else 1,
              _lib.ptr(Z), _lib.ld(Z), float(alpha), _lib.ptr(est))
    return est


def posterior_error_estimate(A, Q, r=config.DEFAULT_PROBES, alpha=config.DEFAULT_ALPHA, seed=0):
    """alpha sqrt(2/pi) max_i ||(I - QQ*) A w_i|| over r fresh Gaussian probes
    (rangefinder.py:65-82); one pass over A (r matvecs)."""
    if r < 1:
        raise ValueError("r must be >= 1")
    if alpha <= 1:
        raise ValueError("alpha must exceed 1")
    op = as_operator(A)
    return float(posterior_error_estimate_dev(op, Q, r, alpha, seed).item())


def adaptive_range_finder(*args, **kwargs):
    raise NotImplementedError(
        "the adaptive (fixed-precision) finder is outside this build's scope (SURVEY.md §8f #1)")


adaptive_range_finder_blocked = adaptive_range_finder
