"""Sparse-plus-low-rank operator on the GPU (configuration 5).

The reference has no sparse code; its extension point for matrix-free A is
the MatVecOperator protocol (core.py:343-380) -- a user subclass with
``_apply`` / ``_apply_adjoint``.  CudaCsrOperator is that subclass on the
device: A = S + L R^T with S in CSR (K6 SpMM kernel) and an optional
implicit low-rank term applied as two skinny GEMMs.  The transpose product
uses a CSR copy of S^T built once at construction (no atomics, so the
product is deterministic).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import MatVecOperator, _as2d, _out, _torch, is_device_array, to_device


def _transpose_csr_device(csr, m, n):
    """CSR of S^T from the CSR of S, on the device (operator construction, not
    the hot path: torch's stable radix sort by column index).  The host
    transpose (scipy) took seconds at config 5's 33.5 M nonzeros and made the
    end-to-end call unmeasurable.  Rows stay ascending within each column (the
    sort is stable), so the result is canonical and the transpose product
    deterministic."""
    torch = _torch()
    rowptr, col, val = csr
    dev = rowptr.device
    nnz = int(col.numel())
    if nnz == 0:
        return (torch.zeros(n + 1, dtype=torch.int64, device=dev), col.clone(), val.clone())
    counts = rowptr[1:] - rowptr[:-1]
    rows = torch.repeat_interleave(torch.arange(m, dtype=torch.int32, device=dev), counts,
                                   output_size=nnz)
    _, perm = torch.sort(col, stable=True)
    t_ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    t_ptr[1:] = torch.cumsum(torch.bincount(col, minlength=n), dim=0)
    return (t_ptr, rows[perm].contiguous(), val[perm].contiguous())


class CudaCsrOperator(MatVecOperator):
    """A = S + L R^T, S sparse (scipy CSR/CSC/COO or (rowptr, col, val, shape))."""

    device_native = True

    def __init__(self, S, L=None, R=None, device=None, host_io=False):
        """host_io: return numpy factors from the range finders / SVD (default:
        CUDA tensors -- the operator lives on the device, like a DenseOperator
        built from a CUDA tensor)."""
        torch = _torch()
        import scipy.sparse as sp
        if isinstance(S, tuple):
            rowptr, col, val, shape = S
            S = sp.csr_matrix((np.asarray(val), np.asarray(col), np.asarray(rowptr)), shape=shape)
        S = sp.csr_matrix(S)
        S.sum_duplicates()
        m, n = S.shape
        super().__init__(m, n)
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.device = dev
        self.S = (torch.from_numpy(S.indptr.astype(np.int64, copy=False)).to(dev),
                  torch.from_numpy(S.indices.astype(np.int32, copy=False)).to(dev),
                  torch.from_numpy(S.data.astype(np.float64, copy=False)).to(dev))
        self.St = _transpose_csr_device(self.S, m, n)
        self.nnz = int(S.nnz)
        self.L = None if L is None else to_device(L, torch.float64, dev.index)
        self.R = None if R is None else to_device(R, torch.float64, dev.index)
        if (self.L is None) != (self.R is None):
            raise ValueError("L and R must be given together")
        if self.L is not None and (self.L.shape[0] != m or self.R.shape[0] != n
                                   or self.L.shape[1] != self.R.shape[1]):
            raise ValueError("low-rank factors do not match the sparse part")
        self.host_io = bool(host_io)
        self.dtype = torch.float64

    def graph_key(self):
        """Data identity for the CUDA-graph cache of repeated steps (factor._run_step)."""
        ptrs = [t.data_ptr() for t in self.S + self.St]
        if self.L is not None:
            ptrs += [self.L.data_ptr(), self.R.data_ptr(), self.L.shape[1]]
        return (self.m, self.n, self.nnz, *ptrs)

    def csr_bytes(self):
        """Bytes of one pass over the CSR data (values, column indices, row pointers)."""
        return self.nnz * (8 + 4) + (self.m + 1) * 8

    def _spmm(self, csr, rows, X, Y, accumulate):
        from . import core
        rowptr, col, val = csr
        if core.PASS_EVENTS is not None:   # bench.py: per-launch timing + bytes model
            torch = _torch()
            s, e = core.timing_event(), core.timing_event()
            torch.cuda.nvtx.range_push("lr_pass")
            s.record()
            self._spmm_launch(rowptr, col, val, rows, X, Y, accumulate)
            e.record()
            torch.cuda.nvtx.range_pop()
            ell = X.shape[1]
            # compulsory bytes: the CSR arrays, X once, Y (read-modify-write
            # when accumulating) -- the schedule-independent HBM lower bound of
            # the product (bench.py adds the cache-capacity-aware bound for
            # random column indices, which is what the gathers actually cost)
            nbytes = (self.csr_bytes() + X.shape[0] * ell * 8
                      + rows * ell * 8 * (2 if accumulate else 1))
            core.PASS_EVENTS.append((s, e, 2 * self.nnz * ell, nbytes, ell))
            return
        self._spmm_launch(rowptr, col, val, rows, X, Y, accumulate)

    def _spmm_launch(self, rowptr, col, val, rows, X, Y, accumulate):
        _lib.call("lr_csr_spmm", _lib.handle(X.device.index), _lib.F64, rows, X.shape[0],
                  X.shape[1], _lib.ptr(rowptr), _lib.ptr(col), _lib.ptr(val), _lib.ptr(X),
                  _lib.ld(X), _lib.ptr(Y), _lib.ld(Y), 1 if accumulate else 0)

    def _lowrank(self, P, Qf, X, Y):
        """Y = P (Qf^T X)  (P: rows x r, Qf: cols x r)."""
        torch = _torch()
        r = P.shape[1]
        Cm = torch.empty((r, X.shape[1]), dtype=torch.float64, device=X.device)
        h = _lib.handle(X.device.index)
        _lib.call("lr_gemm", h, _lib.F64, _lib.OP_T, Qf.shape[0], r, X.shape[1], _lib.ptr(Qf),
                  _lib.ld(Qf), _lib.ptr(X), _lib.ld(X), _lib.ptr(Cm), _lib.ld(Cm))
        _lib.call("lr_gemm", h, _lib.F64, _lib.OP_N, P.shape[0], r, X.shape[1], _lib.ptr(P),
                  _lib.ld(P), _lib.ptr(Cm), _lib.ld(Cm), _lib.ptr(Y), _lib.ld(Y))

    def _run(self, X, adjoint):
        torch = _torch()
        host = not is_device_array(X)
        t = to_device(X, torch.float64, self.device.index)
        t, vec = _as2d(t)
        rows = self.n if adjoint else self.m
        if t.shape[0] != (self.m if adjoint else self.n):
            raise ValueError("dimension mismatch")
        Y = torch.empty((rows, t.shape[1]), dtype=torch.float64, device=t.device)
        acc = False
        if self.L is not None:
            if adjoint:
                self._lowrank(self.R, self.L, t, Y)      # R (L^T Y)
            else:
                self._lowrank(self.L, self.R, t, Y)      # L (R^T X)
            acc = True
        self._spmm(self.St if adjoint else self.S, rows, t, Y, acc)
        Y = Y.reshape(-1) if vec else Y
        return _out(Y, host)

    def _apply(self, X):
        return self._run(X, False)

    def _apply_adjoint(self, Y):
        return self._run(Y, True)
