"""Stage A on the GPU: randomized construction of an orthonormal range basis.

Mirrors the fixed-rank range finders of the reference's
``lowrank.rangefinder`` (/root/reference/pkg/src/lowrank/rangefinder.py)
with identical signatures, validation, pass counting and RangeBasis fields.
The sketch Omega and the estimator probes are drawn ON THE DEVICE from the
reference's Philox streams (gaussian_dev: the same draws as numpy's
Generator(Philox).standard_normal, csrc/gauss.cu); the passes over A, the
orthonormalizations and the estimator tail run on the device and the sample
/ basis panels stay in HBM between steps.  The adaptive (fixed-precision)
finders (Alg 4.2, single-vector and blocked) are here too.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib, config
from .core import (MatVecOperator, _out, _torch, apply_dev, as_operator, cast_dev, gemm,
                   is_device_array, orth_dev, to_device)
from .sketch import SketchSpec, cached_operator, gaussian_dev, gsrft_dev, srft_dev

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


def _adjoint_of_orth(op, Y, ortho_tol):
    """A^H orth(Y).  Inside a speculative step on a device operator the
    second CholeskyQR factor is deferred: orth(Y) = Q1 P2 and A^H Q1 P2 =
    (A^H Q1) P2, an ell x ell product on the n side instead of an m x ell
    panel product (lr_orth_fast_deferred)."""
    from .core import orth_dev_deferred
    d = orth_dev_deferred(Y, ortho_tol) if getattr(op, "device_native", False) else None
    if d is None:
        return apply_dev(op, orth_dev(Y, ortho_tol), adjoint=True)
    Q1, P2 = d
    Z = apply_dev(op, Q1, adjoint=True)
    out = _torch().empty_like(Z)
    gemm(Z, cast_dev(P2, Z.dtype), out)
    return out


def subspace_iteration_range_dev(op, ell, q, seed, ortho_tol=config.GS_DROP_TOL, omega=None):
    """Alg 4.4 on a device operator; returns the device basis.  Same
    products as the reference loop (Q = orth(A Omega); q x [Q~ = orth(A* Q),
    Q = orth(A Q~)]) with each A* Q formed as (A* Q1) P2 (_adjoint_of_orth)."""
    if omega is None:
        omega = _cast_like_op(op, _sketch_dev(op, ell, seed))
    Y = apply_dev(op, omega)
    for _ in range(q):
        Qt = orth_dev(_adjoint_of_orth(op, Y, ortho_tol), ortho_tol)
        Y = apply_dev(op, Qt)
    return orth_dev(Y, ortho_tol)


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
    if isinstance(A, MatVecOperator):
        if not hasattr(A, "array"):
            raise TypeError("fast_range_finder needs a dense matrix")
        host, t, amax = A.host_io, A.array, getattr(A, "amax", None)
    else:
        host = not is_device_array(A)
        t = to_device(A)
        amax = None
    spec = SketchSpec(kind=kind, ell=ell, seed=seed)
    if kind == "srft":
        Y = srft_dev(t, cached_operator("srft", t.shape[1], ell, seed), amax=amax)
    else:
        Y = gsrft_dev(t, cached_operator("gsrft", t.shape[1], ell, seed), amax=amax)
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
    """Estimator probes W (rangefinder.py:78), drawn on the device (gaussian_dev)."""
    Wd = gaussian_dev(op.n, r, seed, stream=_STREAM_PROBE, dtype=_real_of(_op_dtype(op)))
    return _cast_like_op(op, Wd)


def posterior_error_estimate_dev(op, Q, r=config.DEFAULT_PROBES, alpha=config.DEFAULT_ALPHA,
                                 seed=0, W=None):
    """Device estimator; returns a 1-element float64 device tensor."""
    torch = _torch()
    if W is None:
        W = probes_dev(op, r, seed)
    if (getattr(op, "device_native", False) and hasattr(op, "apply_wide")
            and op.dtype == torch.float32 and not W.is_complex()):
        # fp32 operator: the narrow probe pass with exact products and fp64
        # accumulation (the residual is ~1e-5 of |A w| at config 4: below the
        # tensor-core split's rounding), projection in fp64
        Z = op.apply_wide(W)
    else:
        Z = apply_dev(op, W)
    Z = Z.contiguous() if Z.stride(-1) != 1 else Z
    est = torch.empty(1, dtype=torch.float64, device=Z.device)
    Qd = Q if is_device_array(Q) else to_device(Q)
    if Qd.is_complex() and not Z.is_complex():
        # complex (SRFT) basis of a real operator: project in complex
        Z = cast_dev(Z, torch.complex64 if Z.dtype == torch.float32 else torch.complex128)
    Qd = cast_dev(Qd, Z.dtype)
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


_STREAM_ADAPT = 0x61646170      # "adap" (rangefinder.py:121)


def adaptive_range_finder(A, eps, r=config.DEFAULT_PROBES, seed=0, alpha=config.DEFAULT_ALPHA,
                          block=1):
    """Alg 4.2 fixed-precision range finder (rangefinder.py:89-159) on the
    GPU: the basis grows one vector at a time from probe residuals
    y = (I - QQ*) A w, probes drawn in batches of `block` from
    Philox(seed, "adap", index = draws so far); the loop stops once the r
    oldest pending residual norms are <= eps / (alpha sqrt(2/pi)), or with
    `saturated` when the basis reaches min(m, n) columns.  Same reprojection
    (double orthogonalization) and incremental downdate of the pending probes
    as the reference; Q, the pending block and all products stay on the
    device, and each step reads two norms back (the stopping test and the
    new vector's norm)."""
    if eps <= 0:
        raise ValueError("eps must be positive")
    if r < 1:
        raise ValueError("r must be >= 1")
    block = max(int(block), 1)
    torch = _torch()
    op = as_operator(A)
    host = _host_io(A, op)
    m, n = op.shape
    threshold = eps / (alpha * math.sqrt(2.0 / math.pi))
    dt = _op_dtype(op)
    dev = torch.device("cuda", torch.cuda.current_device())
    kmax = min(m, n)
    Qb = torch.empty((m, kmax), dtype=dt, device=dev)
    k = 0
    cap = r + block + 32
    Pm = torch.empty((m, cap), dtype=dt, device=dev)
    head = cnt = 0
    draws = 0
    saturated = False
    code = _lib.dtype_code(dt)
    h = _lib.handle()

    def project(X):
        """X <- X - Q (Q^H X) for the current basis."""
        if k:
            Qk = Qb[:, :k]
            C = torch.empty((k, X.shape[1]), dtype=dt, device=dev)
            gemm(Qk, X, C, adjoint=True)
            T = torch.empty_like(X)
            gemm(Qk, C, T)
            _lib.call("lr_axpy_sub", h, code, X.shape[0], X.shape[1], _lib.ptr(T), _lib.ld(T),
                      _lib.ptr(X), _lib.ld(X))

    def norms(X):
        out = torch.empty(X.shape[1], dtype=torch.float64, device=dev)
        _lib.call("lr_col_sumsq", h, code, X.shape[0], X.shape[1], _lib.ptr(X), _lib.ld(X),
                  _lib.ptr(out))
        return torch.sqrt(out)

    while True:
        while cnt < r:
            W = cast_dev(gaussian_dev(n, block, seed, stream=_STREAM_ADAPT, index=draws,
                                      dtype=_real_of(dt)), dt)
            draws += block
            fresh = apply_dev(op, W)
            if fresh.dim() == 1:
                fresh = fresh.reshape(-1, 1)
            fresh = fresh.contiguous()
            project(fresh)
            if head + cnt + block > cap:                    # compact the pending block
                Pm[:, :cnt] = Pm[:, head:head + cnt].clone()
                head = 0
                if cnt + block > cap:
                    cap = 2 * (cnt + block)
                    P2 = torch.empty((m, cap), dtype=dt, device=dev)
                    P2[:, :cnt] = Pm[:, :cnt]
                    Pm = P2
            Pm[:, head + cnt:head + cnt + block] = fresh
            cnt += block
        if float(norms(Pm[:, head:head + r]).max().item()) <= threshold:
            break
        y = Pm[:, head:head + 1].clone()
        head += 1
        cnt -= 1
        project(y)
        nrm = float(norms(y)[0].item())
        if nrm == 0.0:
            continue
        qk = Qb[:, k:k + 1]
        _lib.call("lr_scale_col", h, code, m, _lib.ptr(y), _lib.ld(y), 1.0 / nrm, _lib.ptr(qk),
                  _lib.ld(qk))
        k += 1
        if k >= kmax:
            saturated = True
            break
        if cnt:
            # pending_i <- pending_i - q (q^H pending_i)
            act = Pm[:, head:head + cnt]
            c = torch.empty((1, cnt), dtype=dt, device=dev)
            gemm(qk, act, c, adjoint=True)
            T = torch.empty((m, cnt), dtype=dt, device=dev)
            gemm(qk, c, T)
            _lib.call("lr_axpy_sub", h, code, m, cnt, _lib.ptr(T), _lib.ld(T), _lib.ptr(act),
                      _lib.ld(act))
    Q = Qb[:, :k].contiguous()
    est = (alpha * math.sqrt(2.0 / math.pi) * float(norms(Pm[:, head:head + min(r, cnt)]).max().item())
           if cnt else 0.0)
    spec = SketchSpec(kind="gaussian", ell=1, seed=seed)
    return RangeBasis(Q=_out(Q, host), samples_used=draws, passes=1, est_error=float(est),
                      spec=spec, saturated=saturated, probe_matvecs=r)


def adaptive_range_finder_blocked(A, eps, r=config.DEFAULT_PROBES, seed=0,
                                  alpha=config.DEFAULT_ALPHA, block=config.ADAPTIVE_BLOCK):
    """Blocked adaptive finder: draws probes in batches of `block`
    (rangefinder.py:162-166)."""
    return adaptive_range_finder(A, eps, r=r, seed=seed, alpha=alpha, block=block)
