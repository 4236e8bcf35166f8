"""Dense kernels and the operator protocol, computed on the GPU.

Mirrors the hot-path part of the reference's ``lowrank.core``
(/root/reference/pkg/src/lowrank/core.py): the MatVecOperator protocol with
its pass / matvec / flop counters (core.py:332-380), a dense operator
(core.py:383-395), double-Gram-Schmidt orthonormalization (core.py:84-115)
and the small SVD with the reference sign convention (core.py:190-230).

Arrays: numpy inputs give numpy outputs (the reference's contract); torch
CUDA tensors stay on the device and give torch tensors.  All arithmetic runs
in liblowrank_b200 (no CPU fallback).  One deliberate difference
(SURVEY.md §7 H9): the reference promotes every input to float64 /
complex128 (core.py:44-47); here float32 / complex64 inputs are computed in
their own precision (with the tensor-core split scheme of DESIGN.md for the
passes over A), float64 / complex128 in theirs, anything else is promoted
to float64 / complex128 like the reference.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import threading
from dataclasses import dataclass

import os

import numpy as np

from . import _lib, config
from ._lib import ConvergenceError, NotPSDError  # noqa: F401  (re-exported, core.py:25-30)


def _torch():
    import torch
    return torch


# ---------------------------------------------------------------------------
# array plumbing

_NP_KEEP = (np.float32, np.float64, np.complex64, np.complex128)


def _np_compute_dtype(dt):
    dt = np.dtype(dt)
    if dt.type in _NP_KEEP:
        return dt
    return np.dtype(np.complex128) if np.issubdtype(dt, np.complexfloating) else np.dtype(np.float64)


def _torch_compute_dtype(t):
    torch = _torch()
    if t.dtype in (torch.float32, torch.float64, torch.complex64, torch.complex128):
        return t.dtype
    return torch.complex128 if t.is_complex() else torch.float64


def is_device_array(x):
    """CUDA tensors stay on the device (device in -> device out); numpy arrays
    and CPU torch tensors are host data (uploaded, results returned as numpy;
    a pinned CPU tensor is uploaded asynchronously at full PCIe rate)."""
    torch = _torch()
    return torch.is_tensor(x) and x.is_cuda


def to_device(x, dtype=None, device=None):
    """numpy / torch -> row-major CUDA tensor (H2D copy for host data)."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    if torch.is_tensor(x):
        t = x
        if t.device != dev:
            t = t.to(dev, non_blocking=True)
        if dtype is not None and t.dtype != dtype:
            t = cast_dev(t, dtype)
    else:
        a = np.asarray(x)
        a = a.astype(_np_compute_dtype(a.dtype), copy=False)
        if dtype is not None:
            want = {torch.float32: np.float32, torch.float64: np.float64,
                    torch.complex64: np.complex64, torch.complex128: np.complex128}[dtype]
            a = a.astype(want, copy=False)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev, non_blocking=False)
    if t.dim() == 2 and t.shape[1] > 1 and t.stride(1) != 1:
        t = t.contiguous()
    if t.dim() == 1 and t.stride(0) != 1:
        t = t.contiguous()
    return t


def _cast_like_dtype(t, dtype):
    """A real draw in the compute dtype of `dtype` (complex operators take
    complex copies; float32 / float64 / complex* kept)."""
    return cast_dev(t, dtype) if t.dtype != dtype else t


def cast_dev(t, dtype):
    """Device dtype conversion with the library's cast kernel (real ->
    complex zero-fills the imaginary part)."""
    if t.dtype == dtype:
        return t
    torch = _torch()
    t2, vec = _as2d(t)
    if t2.shape[1] > 1 and t2.stride(1) != 1:
        t2 = t2.contiguous()
    out = torch.empty(t2.shape, dtype=dtype, device=t2.device)
    if out.numel():
        _lib.call("lr_copy", _lib.handle(t2.device.index), _lib.dtype_code(t2.dtype), _lib.ptr(t2),
                  _lib.ld(t2), _lib.dtype_code(dtype), _lib.ptr(out), _lib.ld(out),
                  t2.shape[0], t2.shape[1], 0)
    return out.reshape(-1) if vec else out


def _stage_host(t):
    """Enqueue the D2H copy of a device tensor into a pinned host buffer
    (torch's caching host allocator: repeated calls reuse the blocks) on the
    current stream; the caller synchronizes once for a batch.  A pageable
    .cpu() runs at a third of the link rate and page-faults a fresh buffer
    every call (13.6 ms for config 2's four factors vs 0.7 ms pinned)."""
    torch = _torch()
    t = t.detach()
    if not t.is_cuda:
        return t
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    if t.numel():
        h.copy_(t, non_blocking=True)
    return h


class HostPrefetch:
    """A device -> pinned-host copy started early on the copy stream, so it
    overlaps the kernels enqueued after it (the basis Q of a randomized SVD
    is final two passes before its factors are)."""

    def __init__(self, t):
        torch = _torch()
        t = t.detach()
        self.src = t
        self.host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        self.event = None
        if t.numel():
            cur = torch.cuda.current_stream(t.device)
            side = _copy_stream(t.device)
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                self.host.copy_(t, non_blocking=True)
                self.event = torch.cuda.Event()
                self.event.record(side)
            t.record_stream(side)

    def numpy(self):
        if self.event is not None:
            self.event.synchronize()
        return self.host.numpy()


def to_host(t):
    return to_hosts(t)[0]


def to_hosts(*ts):
    """Several device tensors -> numpy arrays with one synchronization."""
    torch = _torch()
    hs = [_stage_host(t) for t in ts]
    if any(t.is_cuda for t in ts):
        torch.cuda.current_stream().synchronize()
    return [h.numpy() for h in hs]


def _out(t, host):
    return to_host(t) if host else t


def _outs(host, *ts):
    return to_hosts(*ts) if host else list(ts)


def _as2d(t):
    return (t.reshape(-1, 1), True) if t.dim() == 1 else (t, False)


# ---------------------------------------------------------------------------
# operators (reference core.py:332-402)

@dataclass
class OperatorCounters:
    matvecs: int = 0
    adjoint_matvecs: int = 0
    passes: int = 0
    flops: int = 0

    def reset(self):
        self.matvecs = self.adjoint_matvecs = self.passes = self.flops = 0


class MatVecOperator:
    """Abstract m-by-n linear map with matvec / pass / flop accounting.

    Same protocol as reference core.py:343-380: subclasses implement
    ``_apply`` / ``_apply_adjoint`` on column blocks; ``apply`` counts
    ``cols`` matvecs, one pass and 2*m*n*cols flops.  Operators that set
    ``device_native = True`` receive and return CUDA tensors; others (e.g. a
    user's numpy operator) receive numpy arrays from the GPU pipeline.
    """

    device_native = False

    def __init__(self, m, n):
        self.m = int(m)
        self.n = int(n)
        self.counters = OperatorCounters()

    @property
    def shape(self):
        return (self.m, self.n)

    def _count(self, X, adjoint):
        cols = 1 if X.ndim == 1 else X.shape[1]
        if adjoint:
            self.counters.adjoint_matvecs += cols
        else:
            self.counters.matvecs += cols
        self.counters.passes += 1
        self.counters.flops += 2 * self.m * self.n * cols

    def apply(self, X):
        if not is_device_array(X):
            X = np.asarray(X)
        self._count(X, False)
        return self._apply(X)

    def apply_adjoint(self, Y):
        if not is_device_array(Y):
            Y = np.asarray(Y)
        self._count(Y, True)
        return self._apply_adjoint(Y)

    def _apply(self, X):  # pragma: no cover - abstract
        raise NotImplementedError

    def _apply_adjoint(self, Y):  # pragma: no cover - abstract
        raise NotImplementedError


class DenseOperator(MatVecOperator):
    """GPU-resident dense A: one pass per apply (K1 / K2 kernels).

    Replaces the reference DenseOperator (core.py:383-395).  Construction
    performs the as_matrix checks (2-D, nonempty, finite; core.py:33-50) on
    the device and keeps A in HBM; numpy inputs are uploaded once.
    """

    device_native = True

    # pinned host inputs at least this large are uploaded in row chunks on a
    # copy stream, and the validation and the first pass A*X run chunk by
    # chunk behind the copy (fp64 / complex128: no max|A| needed up front)
    STREAM_MIN_BYTES = 256 << 20
    STREAM_CHUNK_BYTES = 64 << 20
    STREAM_MAX_CHUNKS = 32

    def __init__(self, A, device=None, validate=True):
        torch = _torch()
        host = not is_device_array(A)
        shape = tuple(A.shape) if torch.is_tensor(A) else np.shape(A)
        if len(shape) != 2:
            raise ValueError(f"matrix must be 2-D, got shape {shape}")
        if shape[0] == 0 or shape[1] == 0:
            raise ValueError("matrix must be nonempty")
        self._pending = None
        self.amax = None
        self.host_io = host
        if validate and self._streamable(A):
            super().__init__(*shape)
            self._upload_streamed(A, device)
            if self._array.dtype not in (torch.float64, torch.complex128):
                # fp32 / complex64: join the upload here.  Running the first
                # pass chunk by chunk behind the copy (each chunk scaled by its
                # own max, reduced on the device) measured SLOWER end to end at
                # config 4 (380.0 vs 371.8 ms per call with 32 chunks, 408 ms
                # with 256): the whole-matrix pass after the join costs 5.5 ms,
                # the chunk passes' fixed costs more
                self._finalize()
            return
        t = to_device(A, _torch_compute_dtype(A) if torch.is_tensor(A) else None, device)
        super().__init__(*t.shape)
        self._array = t
        self.code = _lib.dtype_code(t.dtype)
        if validate:
            self.validate()

    @staticmethod
    def _streamable(A):
        torch = _torch()
        return (torch.is_tensor(A) and not A.is_cuda and A.is_pinned() and A.is_contiguous()
                and A.dtype in (torch.float32, torch.float64, torch.complex64, torch.complex128)
                and A.numel() * A.element_size() >= DenseOperator.STREAM_MIN_BYTES)

    def _upload_streamed(self, A, device):
        """H2D in row chunks on a side stream (one event per chunk); the
        as_matrix check of each chunk is enqueued on the current stream
        behind its event, into per-chunk slots read by _finalize()."""
        torch = _torch()
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        t = torch.empty(A.shape, dtype=A.dtype, device=dev)
        self._array = t
        self.code = _lib.dtype_code(t.dtype)
        m, n = A.shape
        # at most ~STREAM_MAX_CHUNKS chunks: every chunk costs a fixed host-side
        # price per pass (a 16 GiB upload in 64 MiB chunks ran 256 chunk passes
        # of 16 row tiles each and became launch-bound: +25 ms)
        cbytes = max(self.STREAM_CHUNK_BYTES, A.numel() * A.element_size() // self.STREAM_MAX_CHUNKS)
        rows = max(128, (cbytes // (n * A.element_size())) // 128 * 128)
        bounds = [(r, min(m, r + rows)) for r in range(0, m, rows)]
        bad = torch.empty(len(bounds), dtype=torch.int64, device=dev)
        res = torch.empty((len(bounds), 2), dtype=torch.float64, device=dev)
        cur = torch.cuda.current_stream(dev)
        side = _copy_stream(dev)
        side.wait_stream(cur)          # t's allocation is ordered before the copies
        chunks = []
        h = _lib.handle(dev.index)
        # float64: the int8-tensor-core digit planes are built chunk by chunk
        # behind the copy too (the whole-matrix prepare would follow the upload)
        oz = None
        if t.dtype == torch.float64 and _ozaki_size_ok(m, n):
            ldp, mp = -(-n // 256) * 256, -(-m // 256) * 256
            try:
                oz = (torch.empty(16 * mp * ldp, dtype=torch.int8, device=dev), ldp,
                      torch.empty(m, dtype=torch.int32, device=dev),
                      torch.zeros(1, dtype=torch.int32, device=dev))
            except torch.cuda.OutOfMemoryError:
                oz = None        # no room for the planes: DMMA passes
        for i, (r0, r1) in enumerate(bounds):
            with torch.cuda.stream(side):
                t[r0:r1].copy_(A[r0:r1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(side)
            cur.wait_event(ev)
            _lib.call("lr_check_finite", h, self.code, r1 - r0, n, _lib.ptr(t[r0:r1]), n,
                      _lib.ptr(bad[i:i + 1]), _lib.ptr(res[i]))
            if oz is not None:
                _lib.call("lr_ozaki_prepare_rows", h, m, n, r0, r1, _lib.ptr(t), n,
                          _lib.ptr(oz[0]), oz[1], _lib.ptr(oz[2]), _lib.ptr(oz[3]))
            chunks.append((r0, r1, ev))
        t.record_stream(side)
        if oz is not None:
            t._lr_ozaki = (t._version, oz)
        self._pending = chunks
        self._checks = (bad, res, A)   # A stays referenced until the copies are done

    def _finalize(self):
        """Join the upload: the current stream waits for the last chunk, and
        the deferred as_matrix result is read (one synchronization)."""
        torch = _torch()
        chunks, self._pending = self._pending, None
        torch.cuda.current_stream(self._array.device).wait_event(chunks[-1][2])
        bad, res, _ = self._checks
        self._checks = None
        oz = getattr(self._array, "_lr_ozaki", None)
        wide = oz[1][3] if oz is not None and oz[1] is not None else torch.zeros(
            1, dtype=torch.int32, device=self._array.device)
        nb, amax, nwide = to_hosts(bad, res[:, 0], wide)
        if int(nb.sum()):
            raise ValueError("matrix contains non-finite entries")
        if oz is not None and int(nwide[0]):
            self._array._lr_ozaki = (self._array._version, None)   # wide rows: DMMA
        self.amax = float(amax.max())
        self._amax_version = self._array._version

    @property
    def array(self):
        if self._pending is not None:
            self._finalize()
        return self._array

    @property
    def device(self):
        return self._array.device

    def validate(self):
        torch = _torch()
        res = torch.empty(2, dtype=torch.float64, device=self.array.device)
        bad = torch.empty(1, dtype=torch.int64, device=self.array.device)
        _lib.call("lr_check_finite", _lib.handle(self.array.device.index), self.code, self.m,
                  self.n, _lib.ptr(self.array), _lib.ld(self.array), _lib.ptr(bad), _lib.ptr(res))
        nb = int(bad.item())
        if nb:
            raise ValueError("matrix contains non-finite entries")
        self.amax = float(res[0].item())
        self._amax_version = self._array._version

    def _refresh(self):
        """max|A| (the power-of-two scale of the fp32 / complex64 tensor-core
        passes) follows in-place modifications of A: a changed version
        counter re-runs the as_matrix check before the next pass."""
        if (self._pending is None and self.amax is not None
                and getattr(self, "_amax_version", self._array._version) != self._array._version):
            self.validate()

    @property
    def dtype(self):
        return self._array.dtype

    def _prep(self, X):
        torch = _torch()
        host = not is_device_array(X)
        dt = self._array.dtype
        if not self._array.is_complex() and (np.iscomplexobj(X) if not torch.is_tensor(X)
                                            else X.is_complex()):
            # real A times a complex block (e.g. the complex SRFT basis of a
            # real matrix): keep X complex, the pass runs on its real view
            dt = torch.complex64 if dt == torch.float32 else torch.complex128
        t = to_device(X, dt, self._array.device.index)
        t, vec = _as2d(t)
        return t, host, vec

    def _run(self, t, adjoint):
        """One pass; a complex t against a real A goes through the real view
        (A^H [Re Im] interleaved == A^H X since A is real)."""
        torch = _torch()
        rows = self.n if adjoint else self.m
        if self._pending is not None and not adjoint and t.dtype == self._array.dtype:
            # first pass of a streamed upload: chunk by chunk behind the copy
            chunks = self._pending
            Y = torch.empty((rows, t.shape[1]), dtype=self._array.dtype, device=t.device)
            cur = torch.cuda.current_stream(t.device)
            for r0, r1, ev in chunks:
                cur.wait_event(ev)
                # (DMMA: digit planes of each chunk view would be rebuilt per call)
                _pass(self._array[r0:r1], t, Y[r0:r1], False, self.amax, allow_ozaki=False)
            self._finalize()
            return Y
        if t.is_complex() and not self.array.is_complex():
            tc = t.contiguous()
            tr = torch.view_as_real(tc).reshape(tc.shape[0], 2 * tc.shape[1])
            Yr = torch.empty((rows, 2 * tc.shape[1]), dtype=self.array.dtype,
                             device=self.array.device)
            _timed_pass(self.array, tr, Yr, adjoint, self.amax)
            return torch.view_as_complex(Yr.reshape(rows, tc.shape[1], 2))
        Y = torch.empty((rows, t.shape[1]), dtype=self.array.dtype, device=self.array.device)
        _timed_pass(self.array, t, Y, adjoint, self.amax)
        return Y

    def _apply(self, X):
        self._refresh()
        t, host, vec = self._prep(X)
        if t.shape[0] != self.n:
            raise ValueError(f"dimension mismatch: A is {self.shape}, X has {t.shape[0]} rows")
        Y = self._run(t, False)
        Y = Y.reshape(-1) if vec else Y
        return _out(Y, host)

    def _apply_adjoint(self, Y):
        self._refresh()
        t, host, vec = self._prep(Y)
        if t.shape[0] != self.m:
            raise ValueError(f"dimension mismatch: A is {self.shape}, Y has {t.shape[0]} rows")
        Z = self._run(t, True)
        Z = Z.reshape(-1) if vec else Z
        return _out(Z, host)


    def apply_wide(self, X):
        """A X for a float32 A with exact products and fp64 accumulation
        (lr_gemm_f64acc, DMMA): one counted pass, fp64 device result.  The
        posterior estimator's narrow pass uses it -- the residual it measures
        sits below the tensor-core split's rounding."""
        torch = _torch()
        A = self.array
        self._refresh()
        t = to_device(X, torch.float32, A.device.index)
        t, vec = _as2d(t)
        self._count(t, False)
        Y = torch.empty((self.m, t.shape[1]), dtype=torch.float64, device=A.device)
        _lib.call("lr_gemm_f64acc", _lib.handle(A.device.index), _lib.OP_N, self.m, self.n,
                  t.shape[1], _lib.ptr(A), _lib.ld(A), _lib.ptr(t), _lib.ld(t), _lib.ptr(Y),
                  _lib.ld(Y))
        return Y.reshape(-1) if vec else Y


CudaDenseOperator = DenseOperator

# Optional per-pass timing (bench.py): a list that receives
# (start_event, end_event, algorithmic_flops, a_bytes, cols) for every pass
# over a dense A, recorded on the launching stream.
PASS_EVENTS = None


_COPY_STREAMS = {}


def _copy_stream(dev):
    torch = _torch()
    st = _COPY_STREAMS.get(dev.index)
    if st is None:
        st = _COPY_STREAMS[dev.index] = torch.cuda.Stream(dev)
    return st


def ozaki_prepare(A):
    """Digit planes of a float64 device matrix for the int8-tensor-core fp64
    passes (lr_ozaki_prepare): (planes, ldp, row_exp, wide_rows); planes holds
    the two shared-memory images of the 8 digit planes (A X and A^T Y tiles),
    16 x MP x ldp bytes (m and n rounded up to 256); wide_rows (device int32)
    counts rows whose nonzero entries span more than 2^32."""
    torch = _torch()
    m, n = A.shape
    ldp = -(-n // 256) * 256          # tiles of 128, padded to pairs (2-SM kernel)
    mp = -(-m // 256) * 256
    planes = torch.empty(16 * mp * ldp, dtype=torch.int8, device=A.device)   # two images
    row_exp = torch.empty(m, dtype=torch.int32, device=A.device)
    wide = torch.zeros(1, dtype=torch.int32, device=A.device)
    _lib.call("lr_ozaki_prepare", _lib.handle(A.device.index), m, n, _lib.ptr(A), _lib.ld(A),
              _lib.ptr(planes), ldp, _lib.ptr(row_exp), _lib.ptr(wide))
    return planes, ldp, row_exp, wide


def ozaki_pass(oz, m, n, X, Y, adjoint):
    """Y = A X (or A^T X) from A's digit planes (lr_gemm_ozaki)."""
    planes, ldp, row_exp = oz[:3]
    _lib.call("lr_gemm_ozaki", _lib.handle(X.device.index), _lib.OP_T if adjoint else _lib.OP_N,
              m, n, X.shape[1], _lib.ptr(planes), ldp, _lib.ptr(row_exp), _lib.ptr(X), _lib.ld(X),
              _lib.ptr(Y), _lib.ld(Y))
    return Y


# Digit planes of a float64 matrix for the int8-tensor-core passes are kept
# on the tensor object itself (attribute _lr_ozaki with its version counter:
# an in-place modification of A rebuilds them), so they live exactly as long
# as A -- and as long as any CUDA graph that replays passes over it through
# the operator holding A.


def _ozaki_wanted(A, X):
    """fp64 passes run on the int8 tensor cores (lr_gemm_ozaki) when that is
    faster than DMMA: the emulated pass costs about the same per 64 output
    columns (128-row x 64-column tiles, 36 digit products) whatever the
    width, the DMMA pass grows with it -- measured crossover near 36
    columns per 64-wide tile (tools/ozaki_probe.py).  LR_OZAKI=0 disables,
    =1 forces it for every fp64 pass."""
    import os
    torch = _torch()
    mode = os.environ.get("LR_OZAKI", "auto")
    if mode == "0" or A.dtype != torch.float64 or A.dim() != 2:
        return False
    ell = X.shape[1]
    if ell < 1 or ell > 256 or A.stride(1) != 1:
        return False
    if mode == "1":
        return True
    m, n = A.shape
    return _ozaki_size_ok(m, n) and ell / -(-ell // 64) >= 40


def _ozaki_size_ok(m, n):
    import os
    return os.environ.get("LR_OZAKI", "auto") != "0" and m >= 1024 and n >= 512


def _ozaki_planes(A):
    """The digit planes of A (built on first use), or None when they do not
    fit in device memory (2 x A's bytes): the passes then stay on DMMA."""
    torch = _torch()
    cached = getattr(A, "_lr_ozaki", None)
    if cached is not None and cached[0] == A._version:
        return cached[1]
    try:
        oz = ozaki_prepare(A)
    except torch.cuda.OutOfMemoryError:
        oz = None
    if oz is not None and int(oz[3].item()):
        # some row's nonzero entries span more than 2^32: the fixed-point
        # digits (relative to the row maximum) would leave its small entries
        # under fp32 precision -- this matrix stays on the DMMA passes
        oz = None
    A._lr_ozaki = (A._version, oz)
    return oz


def _pass(A, X, Y, adjoint, amax, allow_ozaki=True):
    """One pass over A (K1/K2); fp32 / complex64 passes use the tcgen05
    scaled-fp16 split with the operator's max|A| (lr_gemm_scaled); fp64
    passes of enough columns use the int8-tensor-core emulation
    (lr_gemm_ozaki), the others DMMA."""
    oz = _ozaki_planes(A) if allow_ozaki and _ozaki_wanted(A, X) else None
    if oz is not None:
        m, n = A.shape
        ozaki_pass(oz, m, n, X, Y, adjoint)
        return
    code = _lib.dtype_code(A.dtype)
    op = _lib.OP_N if not adjoint else (_lib.OP_C if A.is_complex() else _lib.OP_T)
    m, n = A.shape
    _lib.call("lr_gemm_scaled", _lib.handle(A.device.index), code, op, m, n, X.shape[1],
              _lib.ptr(A), _lib.ld(A), float(-1.0 if amax is None else amax), _lib.ptr(X),
              _lib.ld(X), _lib.ptr(Y), _lib.ld(Y))


def timing_event():
    """CUDA timing event; inside a CUDA-graph capture it becomes an event
    record node (re-recorded by every replay)."""
    torch = _torch()
    return torch.cuda.Event(enable_timing=True,
                            external=bool(torch.cuda.is_current_stream_capturing()))


def _timed_pass(A, X, Y, adjoint, amax=None):
    if PASS_EVENTS is None:
        _pass(A, X, Y, adjoint, amax)
        return
    torch = _torch()
    s, e = timing_event(), timing_event()
    torch.cuda.nvtx.range_push("lr_pass")      # ncu --nvtx-include lr_pass/
    s.record()
    _pass(A, X, Y, adjoint, amax)
    e.record()
    torch.cuda.nvtx.range_pop()
    m, n = A.shape
    mult = 4 if A.is_complex() else 1
    PASS_EVENTS.append((s, e, 2 * mult * m * n * X.shape[1], A.numel() * A.element_size(),
                        X.shape[1]))


class ForeignOperator(MatVecOperator):
    """Adapter for duck-typed operators (e.g. the reference's own
    MatVecOperator subclasses): host numpy in, host numpy out."""

    def __init__(self, op):
        super().__init__(*op.shape)
        self.op = op

    def _apply(self, X):
        return np.asarray(self.op.apply(X))

    def _apply_adjoint(self, Y):
        return np.asarray(self.op.apply_adjoint(Y))


def as_operator(A):
    """Wrap a dense array as DenseOperator; pass operators through
    (reference core.py:398-402)."""
    if isinstance(A, MatVecOperator):
        return A
    if hasattr(A, "apply") and hasattr(A, "apply_adjoint") and hasattr(A, "shape"):
        return ForeignOperator(A)
    return DenseOperator(A)


def apply_dev(op, X, adjoint=False):
    """Apply an operator to a device tensor, whatever kind of operator it is."""
    if op.device_native:
        return op.apply_adjoint(X) if adjoint else op.apply(X)
    Xh = to_host(X)
    R = op.apply_adjoint(Xh) if adjoint else op.apply(Xh)
    return to_device(np.asarray(R), X.dtype, X.device.index)


# ---------------------------------------------------------------------------
# thin wrappers over the C ABI (device tensors in, device tensors out)

def gemm(A, X, Y, adjoint=False):
    """Y = A X (adjoint=False) or Y = A^H X -- one pass over A."""
    code = _lib.dtype_code(A.dtype)
    op = _lib.OP_N if not adjoint else (_lib.OP_C if A.is_complex() else _lib.OP_T)
    m, n = A.shape
    _lib.call("lr_gemm", _lib.handle(A.device.index), code, op, m, n, X.shape[1], _lib.ptr(A),
              _lib.ld(A), _lib.ptr(X), _lib.ld(X), _lib.ptr(Y), _lib.ld(Y))
    return Y


def gemm_dev(A, X, Y):
    """Y = A X for device matrices (the small products U = Q U~ etc.)."""
    return gemm(A, X, Y, adjoint=False)


class _Spec(threading.local):
    status = None


_SPEC = _Spec()


@contextlib.contextmanager
def speculate(status):
    """Run orthonormalizations / small SVDs through the host-sync-free
    speculative kernels, OR-ing their flags into the device int32 `status`
    (see lr_orth_fast).  The caller checks status once at the end and
    re-runs on the synchronous path if any flag is set."""
    prev = _SPEC.status
    _SPEC.status = status
    try:
        yield status
    finally:
        _SPEC.status = prev


def small_svd_from_adjoint(Z):
    """SVD of B = Z^H given Z (c x r, r <= c) -- the layout the adjoint pass
    of direct_svd produces.  Z is consumed (overwritten)."""
    torch = _torch()
    c, r = Z.shape
    if Z.stride(1) != 1 or Z.stride(0) != r:
        Z = Z.contiguous()
    code = _lib.dtype_code(Z.dtype)
    U = torch.empty((r, r), dtype=Z.dtype, device=Z.device)
    S = torch.empty(r, dtype=torch.float64, device=Z.device)
    V = torch.empty((c, r), dtype=Z.dtype, device=Z.device)
    h = _lib.handle(Z.device.index)
    if _SPEC.status is not None:
        _lib.call("lr_small_svd_fast", h, code, r, c, _lib.ptr(Z), _lib.ptr(U), _lib.ptr(S),
                  _lib.ptr(V), _lib.ptr(_SPEC.status))
    else:
        _lib.call("lr_small_svd", h, code, r, c, _lib.ptr(Z), _lib.ptr(U), _lib.ptr(S),
                  _lib.ptr(V))
    return U, S, V


def orth_dev(Y, tol=config.GS_DROP_TOL):
    """Device orthonormalization; returns a (possibly narrower) view."""
    torch = _torch()
    m, ell = Y.shape
    if ell == 0 or m == 0:
        return torch.zeros((m, 0), dtype=Y.dtype, device=Y.device)
    Q = torch.empty((m, ell), dtype=Y.dtype, device=Y.device)
    if _SPEC.status is not None:
        _lib.call("lr_orth_fast", _lib.handle(Y.device.index), _lib.dtype_code(Y.dtype), m, ell,
                  _lib.ptr(Y), _lib.ld(Y), _lib.ptr(Q), _lib.ld(Q), float(tol),
                  _lib.ptr(_SPEC.status))
        return Q
    rank = C.c_int64(0)
    _lib.call("lr_orth", _lib.handle(Y.device.index), _lib.dtype_code(Y.dtype), m, ell,
              _lib.ptr(Y), _lib.ld(Y), _lib.ptr(Q), _lib.ld(Q), float(tol), C.byref(rank))
    r = int(rank.value)
    return Q if r == ell else Q[:, :r]


def orth_dev_deferred(Y, tol=config.GS_DROP_TOL):
    """Speculative CholeskyQR2 without its last panel product
    (lr_orth_fast_deferred): (Q1, P2) with orth(Y) = Q1 P2, or None outside a
    speculative step (the exact path forms Q explicitly)."""
    torch = _torch()
    if _SPEC.status is None:
        return None
    m, ell = Y.shape
    if ell == 0 or m == 0:
        return None
    Q1 = torch.empty((m, ell), dtype=Y.dtype, device=Y.device)
    P2 = torch.empty((ell, ell), dtype=_wide(Y.dtype), device=Y.device)
    _lib.call("lr_orth_fast_deferred", _lib.handle(Y.device.index), _lib.dtype_code(Y.dtype), m,
              ell, _lib.ptr(Y), _lib.ld(Y), _lib.ptr(Q1), _lib.ptr(P2), float(tol),
              _lib.ptr(_SPEC.status))
    return Q1, P2


def orthonormalize_double_gs(Y, tol=config.GS_DROP_TOL):
    """Orthonormalize the columns of Y (replaces reference core.py:84-115).

    Same contract as the reference: columns whose residual after projection
    onto the previously accepted columns is <= tol * ||Y||_F are dropped;
    the result spans a subspace of range(Y); an all-zero Y gives a
    zero-column result.  Computed on the GPU by CholeskyQR2 with an fp64 Gram
    (the Cholesky pivots *are* the residual norms), falling back to shifted
    CholeskyQR3 and then to column-wise CGS2 when a pivot is too small to be
    resolved from the Gram.
    """
    host = not is_device_array(Y)
    t = to_device(Y)
    if t.dim() != 2:
        raise ValueError("Y must be 2-D")
    return _out(orth_dev(t, tol), host)


@dataclass
class SmallSVD:
    """Full SVD B = U @ diag(sigma) @ V*, singular values descending."""

    U: object
    sigma: object
    V: object


def small_svd_dev(B):
    """Thin SVD of a device matrix B (r x c); returns device tensors."""
    torch = _torch()
    r, c = B.shape
    code = _lib.dtype_code(B.dtype)
    h = _lib.handle(B.device.index)
    if r == 0 or c == 0:
        k = min(r, c)
        return (torch.zeros((r, k), dtype=B.dtype, device=B.device),
                torch.zeros(k, dtype=torch.float64, device=B.device),
                torch.zeros((c, k), dtype=B.dtype, device=B.device))
    if r <= c:
        Bh = torch.empty((c, r), dtype=B.dtype, device=B.device)
        _lib.call("lr_copy", h, code, _lib.ptr(B), _lib.ld(B), code, _lib.ptr(Bh), _lib.ld(Bh),
                  c, r, 1)
        U = torch.empty((r, r), dtype=B.dtype, device=B.device)
        S = torch.empty(r, dtype=torch.float64, device=B.device)
        V = torch.empty((c, r), dtype=B.dtype, device=B.device)
        _lib.call("lr_small_svd", h, code, r, c, _lib.ptr(Bh), _lib.ptr(U), _lib.ptr(S),
                  _lib.ptr(V))
        return U, S, V
    # tall B: SVD of B^H (c x r, c < r), B = V' S U'^H
    Bc = B.contiguous().clone()
    U1 = torch.empty((c, c), dtype=B.dtype, device=B.device)
    S = torch.empty(c, dtype=torch.float64, device=B.device)
    V1 = torch.empty((r, c), dtype=B.dtype, device=B.device)
    _lib.call("lr_small_svd", h, code, c, r, _lib.ptr(Bc), _lib.ptr(U1), _lib.ptr(S),
              _lib.ptr(V1))
    U, V = V1, U1
    _lib.call("lr_sign_fix", h, code, r, c, c, _lib.ptr(U), _lib.ld(U), _lib.ptr(V), _lib.ld(V))
    return U, S, V


def small_svd(B):
    """Thin SVD with the reference's deterministic sign convention
    (core.py:199-230): sigma descending; the first entry of each left
    vector with |u| > 1e-10 max|u| is real positive and V absorbs the
    phase.  A non-converging iteration raises ConvergenceError."""
    host = not is_device_array(B)
    t = to_device(B)
    if t.dim() != 2:
        raise ValueError("B must be 2-D")
    U, S, V = small_svd_dev(t)
    U, S, V = _outs(host, U, S, V)
    return SmallSVD(U=U, sigma=S, V=V)


# ---------------------------------------------------------------------------
# small Hermitian eigendecomposition (reference core.py:233-246)

def _wide(dtype):
    torch = _torch()
    return torch.complex128 if dtype in (torch.complex64, torch.complex128) else torch.float64


def small_eig_hermitian_dev(B):
    """Eigenpairs of the Hermitian part of a device matrix B (k x k):
    (V, lam), lam float64 ordered by descending |lam| (ties: descending lam).

    Computed as the SVD of the shifted SPD matrix (B + B^H)/2 + s I,
    s = 2 ||(B + B^H)/2||_F (condition number <= 3), by the K4 small-SVD
    kernels: lam = sigma - s, absolute accuracy O(u ||B||) like LAPACK eigh."""
    torch = _torch()
    k = B.shape[0]
    if B.dim() != 2 or B.shape[1] != k:
        raise ValueError("small_eig_hermitian requires a square matrix")
    wd = _wide(B.dtype)
    if k == 0:
        return (torch.zeros((0, 0), dtype=wd, device=B.device),
                torch.zeros(0, dtype=torch.float64, device=B.device))
    Bw = cast_dev(B, wd).contiguous()
    code = _lib.dtype_code(wd)
    h = _lib.handle(B.device.index)
    H = torch.empty((k, k), dtype=wd, device=B.device)
    out2 = torch.zeros(2, dtype=torch.float64, device=B.device)
    _lib.call("lr_herm_prep", h, code, k, _lib.ptr(Bw), _lib.ld(Bw), _lib.ptr(H), 2.0, 0,
              _lib.ptr(out2))
    U, S, _ = small_svd_dev(H)
    lam = torch.empty(k, dtype=torch.float64, device=B.device)
    V = torch.empty((k, k), dtype=wd, device=B.device)
    _lib.call("lr_eig_finish", h, code, k, _lib.ptr(S), _lib.ptr(out2), _lib.ptr(U.contiguous()),
              _lib.ptr(lam), _lib.ptr(V))
    return V, lam


def small_eig_hermitian(B):
    """Eigendecomposition of a Hermitian matrix, symmetrized internally
    (replaces reference core.py:233-246).  Returns (V, lam): real lam by
    descending magnitude (equal magnitudes in descending value), orthonormal
    V."""
    host = not is_device_array(B)
    t = to_device(B)
    if t.dim() != 2 or t.shape[0] != t.shape[1]:
        raise ValueError("small_eig_hermitian requires a square matrix")
    V, lam = small_eig_hermitian_dev(t)
    return _out(V, host), _out(lam, host)
