"""Row-block streaming of stored matrices and the one-pass two-sided sketch.

Mirrors the hot-path part of the reference's ``lowrank.io``
(/root/reference/pkg/src/lowrank/io.py): the ``LRKMAT00`` binary container
(io.py:35, 178-204), ``RowBlockStream`` / ``stream_row_blocks``
(io.py:319-356), ``accumulate_two_sided_samples`` (io.py:364-388),
``streamed_sample_bundle`` (io.py:391-404) and ``in_memory_sample_bundle``
(io.py:407-430).  This is the route to matrices larger than HBM (SURVEY.md
§8f #2): A is read once, block by block, and both sketches are accumulated on
the GPU,

    Y[rows]  = block Omega           (lr_gemm, one pass over the block)
    Y~      += block^H Omega~[rows]  (lr_gemm adjoint + lr_axpy_add)

with Omega = gaussian_matrix(n, ell, seed) and Omega~ = gaussian_matrix(m,
ell~, seed + 1) drawn on the device from the reference's Philox streams.
Blocks read from a file are staged through pinned host buffers and copied on
a side stream, so the copy of block i+1 overlaps the products of block i;
only two blocks are resident at a time.  The arithmetic order is fixed by
the block sequence, so two runs over the same blocks agree bitwise, and a
streamed run equals an in-memory run with the same block size bitwise (the
reference's contract, io.py:367-371, tests/test_io.py:187-198).

File parsing (header, magic, truncation checks) is host I/O and follows the
reference; everything numeric runs in liblowrank_b200.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import _torch, is_device_array, to_device, to_hosts

_MAGIC = b"LRKMAT00"
_HEADER = 8 + 24


class MatrixFormatError(ValueError):
    """A file failed to parse (reference io.py:38-39)."""


class StreamError(IOError):
    """A row-block stream hit a truncated or inconsistent source (io.py:42-43)."""


# ---------------------------------------------------------------------------
# binary container (io.py:178-204)

def write_matrix_binary(A, path):
    """LRKMAT00 writer: magic, int64 {complex flag, m, n}, then the entries
    row-major as <f8 or <c16 (reference io.py:178-188, which promotes to
    float64 / complex128)."""
    A = np.asarray(A.cpu() if hasattr(A, "cpu") else A)
    if A.ndim != 2 or A.size == 0:
        raise ValueError("matrix must be 2-D and nonempty")
    if not np.all(np.isfinite(A)):
        raise ValueError("matrix contains non-finite entries")
    cplx = np.iscomplexobj(A)
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        np.asarray([1 if cplx else 0, A.shape[0], A.shape[1]], dtype="<i8").tofile(fh)
        np.ascontiguousarray(A).astype("<c16" if cplx else "<f8").tofile(fh)


def read_header(path):
    """(field code, m, n) of a LRKMAT00 file; MatrixFormatError on a bad
    magic or a truncated header (io.py:191-197)."""
    with open(path, "rb") as fh:
        magic = fh.read(8)
        if magic != _MAGIC:
            raise MatrixFormatError(f"{path}: bad magic {magic!r}")
        head = np.fromfile(fh, dtype="<i8", count=3)
    if head.size != 3:
        raise MatrixFormatError(f"{path}: truncated header")
    code, m, n = (int(x) for x in head)
    return code, m, n


def read_matrix_binary(path, device=None):
    """Read a LRKMAT00 matrix (io.py:191-204).  device=None returns the
    reference's numpy array; device="cuda" (or a device index) streams the
    data section straight into HBM through pinned staging buffers and runs
    the as_matrix finiteness check there (lr_check_finite)."""
    code, m, n = read_header(path)
    if device is None:
        dtype = "<c16" if code == 1 else "<f8"
        with open(path, "rb") as fh:
            fh.seek(_HEADER)
            data = np.fromfile(fh, dtype=dtype, count=m * n)
        if data.size != m * n:
            raise MatrixFormatError(f"{path}: truncated data section")
        data = data.reshape(m, n)
        if data.size == 0:
            raise ValueError("matrix must be nonempty")
        if not np.all(np.isfinite(data)):
            raise ValueError(f"{path}: matrix contains non-finite entries")
        return data
    torch = _torch()
    dev = None if isinstance(device, str) else int(device)
    stream = RowBlockStream(path, max(1, (64 << 20) // (n * (16 if code == 1 else 8))))
    out = None
    for row, blk in stream.device_blocks(device=dev, raise_format=True):
        if out is None:
            out = torch.empty((m, n), dtype=blk.dtype, device=blk.device)
        out[row:row + blk.shape[0]].copy_(blk)
    if out is None:
        raise ValueError("matrix must be nonempty")
    bad = torch.empty(1, dtype=torch.int64, device=out.device)
    res = torch.empty(2, dtype=torch.float64, device=out.device)
    _lib.call("lr_check_finite", _lib.handle(out.device.index), _lib.dtype_code(out.dtype), m, n,
              _lib.ptr(out), _lib.ld(out), _lib.ptr(bad), _lib.ptr(res))
    if int(bad.item()):
        raise ValueError(f"{path}: matrix contains non-finite entries")
    return out


# ---------------------------------------------------------------------------
# row-block streaming (io.py:319-356)

@dataclass
class RowBlockStream:
    """Iterator over consecutive row blocks of a stored binary matrix.

    Iterating yields (row_offset, numpy block) like the reference;
    device_blocks() yields (row_offset, CUDA tensor) with the file reads,
    pinned staging and host-to-device copies of the next block overlapped
    with whatever the caller enqueues on the current stream."""

    path: str
    block_rows: int

    def __post_init__(self):
        if self.block_rows < 1:
            raise ValueError("block_rows must be >= 1")
        with open(self.path, "rb") as fh:
            if fh.read(8) != _MAGIC:
                raise MatrixFormatError(f"{self.path}: bad magic")
            head = np.fromfile(fh, dtype="<i8", count=3)
        if head.size != 3:
            raise MatrixFormatError(f"{self.path}: truncated header")
        self.field_code, self.m, self.n = (int(x) for x in head)
        self.cursor = 0

    @property
    def shape(self):
        return (self.m, self.n)

    @property
    def np_dtype(self):
        return np.dtype("<c16" if self.field_code == 1 else "<f8")

    def __iter__(self):
        dtype = self.np_dtype
        with open(self.path, "rb") as fh:
            fh.seek(_HEADER)
            row = 0
            while row < self.m:
                rows = min(self.block_rows, self.m - row)
                data = np.fromfile(fh, dtype=dtype, count=rows * self.n)
                if data.size != rows * self.n:
                    raise StreamError(
                        f"{self.path}: stream truncated at row block starting {row}")
                self.cursor = row + rows
                yield row, data.reshape(rows, self.n)
                row += rows

    def device_blocks(self, device=None, raise_format=False):
        """Yield (row, CUDA tensor) blocks: the file is read with readinto
        into one of two pinned buffers, copied on a side stream, and the
        current stream waits on the copy's event; the buffer is reused two
        blocks later, after the copy that read it has completed."""
        torch = _torch()
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        tdt = torch.complex128 if self.field_code == 1 else torch.float64
        es = 16 if self.field_code == 1 else 8
        cap = min(self.block_rows, self.m) * self.n
        pins = [torch.empty(cap, dtype=tdt, pin_memory=True) for _ in range(2)]
        done = [None, None]
        cur = torch.cuda.current_stream(dev)
        side = torch.cuda.Stream(dev)
        with open(self.path, "rb") as fh:
            fh.seek(_HEADER)
            row, i = 0, 0
            while row < self.m:
                rows = min(self.block_rows, self.m - row)
                slot = i & 1
                if done[slot] is not None:
                    done[slot].synchronize()            # the copy that read this buffer
                buf = pins[slot][:rows * self.n]
                view = buf.view(torch.uint8).numpy()
                got = fh.readinto(memoryview(view))
                if got != rows * self.n * es:
                    err = MatrixFormatError if raise_format else StreamError
                    raise err(f"{self.path}: stream truncated at row block starting {row}")
                dst = torch.empty((rows, self.n), dtype=tdt, device=dev)
                side.wait_stream(cur)                   # dst's allocation is ordered first
                with torch.cuda.stream(side):
                    dst.copy_(buf.view(rows, self.n), non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(side)
                done[slot] = ev
                cur.wait_event(ev)
                dst.record_stream(cur)
                self.cursor = row + rows
                yield row, dst
                row += rows
                i += 1


def stream_row_blocks(path, block_rows):
    """Open a stored matrix for one-pass row-block traversal (io.py:355-356)."""
    return RowBlockStream(path=path, block_rows=block_rows)


# ---------------------------------------------------------------------------
# one-pass two-sided accumulation (io.py:364-388)

def _wide_of(dt_np_or_torch):
    torch = _torch()
    if torch.is_tensor(dt_np_or_torch):
        return torch.complex128 if dt_np_or_torch.is_complex() else torch.float64
    return torch.complex128 if np.iscomplexobj(dt_np_or_torch) else torch.float64


def accumulate_two_sided_samples_dev(blocks, m, n, ell, ell_tilde, seed, device=None):
    """Device accumulation; returns device (Omega, Omega_t, Y, Yt)."""
    torch = _torch()
    from .core import gemm
    from .sketch import gaussian_dev
    dev = torch.cuda.current_device() if device is None else device
    Omega = gaussian_dev(n, ell, seed, device=dev)
    Omega_t = gaussian_dev(m, ell_tilde, seed + 1, device=dev)
    Y = Yt = None
    total = 0
    h = _lib.handle(dev)
    T = None
    for row, block in blocks:
        if Y is None:
            wd = _wide_of(block)
            Y = torch.zeros((m, ell), dtype=wd, device=f"cuda:{dev}")
            Yt = torch.zeros((n, ell_tilde), dtype=wd, device=f"cuda:{dev}")
            T = torch.empty((n, ell_tilde), dtype=wd, device=f"cuda:{dev}")
            Om = Omega.to(wd) if wd == torch.complex128 else Omega
            Omt = Omega_t.to(wd) if wd == torch.complex128 else Omega_t
        b = to_device(block, Y.dtype, dev)
        if b.dim() == 1:
            b = b.reshape(1, -1)
        rows = b.shape[0]
        if b.shape[1] != n or row + rows > m:
            raise StreamError(f"block at row {row} does not fit a {m} x {n} matrix")
        gemm(b, Om, Y[row:row + rows])                       # Y[rows] = block Omega
        gemm(b, Omt[row:row + rows], T, adjoint=True)        # T = block^H Omega~[rows]
        _lib.call("lr_axpy_add", h, _lib.dtype_code(Yt.dtype), n, ell_tilde, _lib.ptr(T),
                  _lib.ld(T), _lib.ptr(Yt), _lib.ld(Yt))
        total += rows
    if total != m:
        raise StreamError(f"stream delivered {total} rows, expected {m}")
    return Omega, Omega_t, Y, Yt


def accumulate_two_sided_samples(blocks, m, n, ell, ell_tilde, seed):
    """Y = A Omega and Y~ = A* Omega~ from one traversal of row blocks
    (reference io.py:364-388).  `blocks` yields (row_offset, block) pairs
    covering the matrix once, in order; numpy blocks give numpy outputs,
    CUDA blocks stay on the device."""
    it = iter(blocks)
    first = next(it, None)
    if first is None:
        raise StreamError(f"stream delivered 0 rows, expected {m}")
    host = not is_device_array(first[1])

    def chain():
        yield first
        yield from it

    out = accumulate_two_sided_samples_dev(chain(), m, n, ell, ell_tilde, seed)
    return tuple(to_hosts(*out)) if host else out


def streamed_sample_bundle(stream, ell, ell_tilde=None, seed=0, rank=None, device_blocks=True):
    """Two-sided SampleBundle accumulated from a RowBlockStream in one pass
    (io.py:391-404): the blocks are streamed to the GPU (pinned, overlapped
    copies), the bases computed there; numpy outputs like the reference."""
    from .factor import SampleBundle, _basis_from_samples_dev
    if ell_tilde is None:
        ell_tilde = ell
    m, n = stream.shape
    blocks = stream.device_blocks() if device_blocks else iter(stream)
    Omega, Omega_t, Y, Yt = accumulate_two_sided_samples_dev(blocks, m, n, ell, ell_tilde, seed)
    Q, choice = _basis_from_samples_dev(Y, rank)
    Qt, _ = _basis_from_samples_dev(Yt, rank)
    Omega, Y, Q, Omega_t, Yt, Qt = to_hosts(Omega, Y, Q, Omega_t, Yt, Qt)
    return SampleBundle(Omega=Omega, Y=Y, Q=Q, Omega_tilde=Omega_t, Y_tilde=Yt, Q_tilde=Qt,
                        q_choice=choice, seed=seed)


def in_memory_sample_bundle(A, ell, ell_tilde=None, seed=0, rank=None, block_rows=None):
    """Two-sided bundle from an in-memory matrix via the same accumulation
    (io.py:407-430); with block_rows set the arithmetic order matches a
    streamed run with the same block size bit for bit."""
    from .factor import SampleBundle, _basis_from_samples_dev
    host = not is_device_array(A)
    if host:
        An = np.asarray(A)
        if An.ndim != 2 or An.size == 0:
            raise ValueError("matrix must be 2-D and nonempty")
        if not np.all(np.isfinite(An)):
            raise ValueError("matrix contains non-finite entries")
        A = An.astype(np.complex128 if np.iscomplexobj(An) else np.float64, copy=False)
    if ell_tilde is None:
        ell_tilde = ell
    m, n = A.shape
    step = block_rows or m

    def blocks():
        for row in range(0, m, step):
            yield row, A[row:row + step]

    Omega, Omega_t, Y, Yt = accumulate_two_sided_samples_dev(blocks(), m, n, ell, ell_tilde, seed)
    Q, choice = _basis_from_samples_dev(Y, rank)
    Qt, _ = _basis_from_samples_dev(Yt, rank)
    outs = (Omega, Y, Q, Omega_t, Yt, Qt)
    if host:
        outs = to_hosts(*outs)
    Omega, Y, Q, Omega_t, Yt, Qt = outs
    return SampleBundle(Omega=Omega, Y=Y, Q=Q, Omega_tilde=Omega_t, Y_tilde=Yt, Q_tilde=Qt,
                        q_choice=choice, seed=seed)


__all__ = ["MatrixFormatError", "StreamError", "RowBlockStream", "accumulate_two_sided_samples",
           "in_memory_sample_bundle", "read_header", "read_matrix_binary", "stream_row_blocks",
           "streamed_sample_bundle", "write_matrix_binary"]
