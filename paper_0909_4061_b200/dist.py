"""Row-sharded randomized SVD over several GPUs.

A is split by rows over the ranks (rank r holds rows [r0, r1)).  The passes
need exactly two kinds of exchange, both all-reduces over NVLink (NCCL via
torch.distributed):
  * A X: local rows of Y = A_r X, no communication (X replicated);
  * A^H Y: Z = sum_r A_r^H Y_r -- an all-reduce of the n x ell partials;
  * orthonormalization of the row-sharded panel Y: G = sum_r Y_r^H Y_r -- an
    all-reduce of the ell x ell Gram; the Cholesky (and its rank decision) is
    computed redundantly on every rank from the identical G, Q_r = Y_r P.
The small SVD of direct_svd is replicated (Z is replicated after its
all-reduce) and U_r = Q_r U~ is local.  The sketch Omega / probes W are drawn
identically on every rank (same Philox stream, reference sketch.py:32-42).

This mirrors the reference's only decomposed pass -- the row-block sum of
accumulate_two_sided_samples (io.py:364-388) -- with the block sum turned
into an all-reduce.  The orchestration is written against a small backend
interface: GpuBackend (liblowrank_b200 kernels, torch CUDA tensors) is the
product; tests/ drive the same host logic with a numpy backend over gloo.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from . import _lib, config

U64 = 1.1102230246251565e-16


class Comm:
    """Sum / max all-reduce over a torch.distributed group (NCCL or gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allreduce(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def allreduce_max(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t

    def allgather_rows(self, t, total):
        """Row shards (row_range split of `total` rows) -> the full matrix on
        every rank (the n-side panel before a pass A_r X, config 5)."""
        if self.world == 1:
            return t
        import torch
        sizes = [row_range(total, r, self.world) for r in range(self.world)]
        mx = max(b - a for a, b in sizes)
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[:t.shape[0]] = t
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[:b - a] for p, (a, b) in zip(parts, sizes)], dim=0).contiguous()

    def reduce_scatter_rows(self, t, total):
        """Full-size partials (total x c, one per rank) -> this rank's rows of
        their sum (the n-side result of A^H Y over row-sharded A, config 5):
        reduce-scatter over NCCL, all-reduce + slice where the backend has no
        reduce-scatter (gloo)."""
        if self.world == 1:
            return t
        import torch
        a, b = row_range(total, self.rank, self.world)
        sizes = [row_range(total, r, self.world) for r in range(self.world)]
        even = all(bb - aa == b - a for aa, bb in sizes)
        if even and self.dist.get_backend(self.group) == "nccl":
            out = torch.empty((b - a,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            self.dist.reduce_scatter_tensor(out, t.contiguous(), op=self.dist.ReduceOp.SUM,
                                            group=self.group)
            return out
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t[a:b].contiguous()


class GpuBackend:
    """Kernels of liblowrank_b200 on torch CUDA tensors (the product path)."""

    def __init__(self):
        import torch
        self.torch = torch

    # --- passes over the local rows of A
    def pass_n(self, A, X, amax=None):
        from .core import _timed_pass
        Y = self.torch.empty((A.shape[0], X.shape[1]), dtype=A.dtype, device=A.device)
        _timed_pass(A, X, Y, False, amax)
        return Y

    def pass_t(self, A, Y, amax=None):
        from .core import _timed_pass
        Z = self.torch.empty((A.shape[1], Y.shape[1]), dtype=A.dtype, device=A.device)
        _timed_pass(A, Y, Z, True, amax)
        return Z

    def srft(self, A, ell, seed):
        from .sketch import srft_dev, srft_operator
        return srft_dev(A, srft_operator(A.shape[1], ell, seed))

    # --- passes of a row-block operator A_r (m_r x n), e.g. CudaCsrOperator
    def op_n(self, op, X):
        return op.apply(X)

    def op_t(self, op, Y):
        return op.apply_adjoint(Y)

    # --- panel kernels
    def gram(self, Y):
        torch = self.torch
        ell = Y.shape[1]
        G = torch.empty((ell, ell), dtype=_lib.wide_torch(_lib.dtype_code(Y.dtype)),
                        device=Y.device)
        _lib.call("lr_gram", _lib.handle(Y.device.index), _lib.dtype_code(Y.dtype), Y.shape[0],
                  ell, _lib.ptr(Y), _lib.ld(Y), _lib.ptr(G))
        return G

    def chol(self, G, drop_tol, unres_rel, shift_coef):
        """(P, R, rank, unresolved, bad) -- replicated on every rank."""
        torch = self.torch
        ell = G.shape[0]
        P = torch.empty_like(G)
        R = torch.empty_like(G)
        info = torch.zeros(4, dtype=torch.int32, device=G.device)
        code = _lib.C128 if G.is_complex() else _lib.F64
        _lib.call("lr_chol_drop", _lib.handle(G.device.index), code, ell, _lib.ptr(G),
                  float(drop_tol), float(unres_rel), float(shift_coef), _lib.ptr(P), _lib.ptr(R),
                  _lib.ptr(info))
        inf = info.cpu().tolist()
        return P, R, inf[0], inf[1], inf[2]

    def chol_fast(self, G, drop_tol, unres_rel, near_thr, status):
        """Host-sync-free Cholesky: P only; decisions ORed into `status`
        (device int32: 1 unresolved, 2 dropped, 4 non-finite)."""
        torch = self.torch
        ell = G.shape[0]
        P = torch.empty_like(G)
        R = torch.empty_like(G)
        info = torch.zeros(4, dtype=torch.int32, device=G.device)
        code = _lib.C128 if G.is_complex() else _lib.F64
        _lib.call("lr_chol_drop_fast", _lib.handle(G.device.index), code, ell, _lib.ptr(G),
                  float(drop_tol), float(unres_rel), 0.0, float(near_thr), _lib.ptr(P),
                  _lib.ptr(R), _lib.ptr(info), _lib.ptr(status))
        return P

    def new_status(self, like):
        return self.torch.zeros(1, dtype=self.torch.int32, device=like.device)

    def like(self, op):
        """A device tensor of the operator's dtype / device (draw template)."""
        return self.torch.empty(0, dtype=op.dtype, device=op.device)

    def status_value(self, status):
        return int(status.item())

    def speculate(self, status):
        from .core import speculate
        return speculate(status)

    def apply(self, Y, P, ncols):
        """Y @ P[:, :ncols] in the panel precision."""
        from .core import cast_dev, gemm_dev
        torch = self.torch
        Pc = cast_dev(P[:, :ncols].contiguous(), Y.dtype)
        out = torch.empty((Y.shape[0], ncols), dtype=Y.dtype, device=Y.device)
        gemm_dev(Y, Pc, out)
        return out

    def matmul(self, A, B):
        from .core import gemm_dev
        out = self.torch.empty((A.shape[0], B.shape[1]), dtype=A.dtype, device=A.device)
        gemm_dev(A, B, out)
        return out

    def adj_matmul(self, A, B):
        """A^H B (small result, reduction over the local rows)."""
        from .core import gemm
        out = self.torch.empty((A.shape[1], B.shape[1]), dtype=A.dtype, device=A.device)
        gemm(A, B, out, adjoint=True)
        return out

    def sub_(self, Z, T):
        _lib.call("lr_axpy_sub", _lib.handle(Z.device.index), _lib.dtype_code(Z.dtype),
                  Z.shape[0], Z.shape[1], _lib.ptr(T), _lib.ld(T), _lib.ptr(Z), _lib.ld(Z))
        return Z

    def colsumsq(self, Z):
        torch = self.torch
        out = torch.empty(Z.shape[1], dtype=torch.float64, device=Z.device)
        _lib.call("lr_col_sumsq", _lib.handle(Z.device.index), _lib.dtype_code(Z.dtype),
                  Z.shape[0], Z.shape[1], _lib.ptr(Z), _lib.ld(Z), _lib.ptr(out))
        return out

    def small_svd(self, Z):
        from .core import small_svd_from_adjoint
        return small_svd_from_adjoint(Z.contiguous())

    def gaussian(self, n, ell, seed, stream, like):
        from .sketch import gaussian_dev
        torch = self.torch
        real = torch.float32 if like.dtype in (torch.float32, torch.complex64) else torch.float64
        from .core import cast_dev
        return cast_dev(gaussian_dev(n, ell, seed, stream=stream, dtype=real,
                                     device=like.device.index), like.dtype)

    def zeros_like_rows(self, Y, ncols):
        return self.torch.zeros((Y.shape[0], ncols), dtype=Y.dtype, device=Y.device)

    def zeros_rows(self, rows, ncols, like):
        return self.torch.zeros((rows, ncols), dtype=like.dtype, device=like.device)

    def empty_sigma(self, like):
        return self.torch.zeros(0, dtype=self.torch.float64, device=like.device)

    def trace(self, G):
        return float(self.torch.diagonal(G).real.sum().item())

    def column(self, Y, j):
        from .core import cast_dev
        return cast_dev(Y[:, j:j + 1], Y.dtype)

    def set_column(self, Q, j, w, inv):
        dst = Q[:, j:j + 1]
        _lib.call("lr_scale_col", _lib.handle(Q.device.index), _lib.dtype_code(Q.dtype),
                  Q.shape[0], _lib.ptr(w), _lib.ld(w), float(inv), _lib.ptr(dst), _lib.ld(dst))

    def to_scalar(self, t):
        return float(t.max().item())


_STREAM_GAUSS = 0x67617573
_STREAM_PROBE = 0x70726F62


def dist_orth(Y, comm, be, tol=config.GS_DROP_TOL):
    """Orthonormalize a row-sharded panel (replaces orthonormalize_double_gs,
    reference core.py:84-115, for A split by rows).

    Fast path: CholeskyQR2 on the all-reduced Gram; the Cholesky pivots are
    the squared Gram-Schmidt residuals, so the reference's drop rule
    (residual <= tol ||Y||_F, core.py:104-106) is applied to the global
    pivots identically on every rank.  When a pivot is too small to be
    resolved from the Gram (4 ell u relative), the column-wise CGS2 of the
    reference runs with one all-reduce per projection / norm.  Returns the
    local rows of Q (every rank gets the same column count)."""
    m_local, ell = Y.shape
    unres = 4.0 * ell * U64
    G = comm.allreduce(be.gram(Y))
    P, _, rank, unresolved, bad = be.chol(G, tol, unres, 0.0)
    if bad:
        raise ValueError("orthonormalize: non-finite entries in the sample matrix")
    if rank == 0:
        return be.zeros_like_rows(Y, 0)
    if unresolved == 0:
        Q1 = be.apply(Y, P, rank)
        G2 = comm.allreduce(be.gram(Q1))
        P2, _, rank2, unres2, bad2 = be.chol(G2, tol, unres, 0.0)
        if rank2 == rank and unres2 == 0 and bad2 == 0:
            return be.apply(Q1, P2, rank)
    return dist_cgs2(Y, comm, be, tol, math.sqrt(be.trace(G)))


def dist_orth_fast(Y, comm, be, status, tol=config.GS_DROP_TOL):
    """Speculative row-sharded CholeskyQR2 (no host synchronization): the
    drop / resolvability decisions of the exact path are evaluated on the
    device (identically on every rank -- the Gram is all-reduced) and ORed
    into `status`; a nonzero status at the end of the step sends every rank
    back to the exact path (dist_orth)."""
    ell = Y.shape[1]
    unres = 4.0 * ell * U64
    G = comm.allreduce(be.gram(Y))
    Q1 = be.apply(Y, be.chol_fast(G, tol, unres, 0.0, status), ell)
    G2 = comm.allreduce(be.gram(Q1))
    near = 1e-4 if str(Y.dtype).endswith(("float32", "complex64")) else 1e-8
    return be.apply(Q1, be.chol_fast(G2, tol, unres, near, status), ell)


def dist_cgs2(Y, comm, be, tol, fro):
    """Column-wise classical Gram-Schmidt with one re-orthogonalization
    (reference core.py:99-114) on a row-sharded panel."""
    m_local, ell = Y.shape
    Q = be.zeros_like_rows(Y, ell)
    kept = 0

    def project(w):
        if kept:
            Qk = Q[:, :kept]
            c = comm.allreduce(be.adj_matmul(Qk, w))
            be.sub_(w, be.matmul(Qk, c))

    def norm(w):
        return math.sqrt(be.to_scalar(comm.allreduce(be.colsumsq(w))))

    for j in range(ell):
        w = be.column(Y, j)
        project(w)
        n1 = norm(w)
        if n1 <= tol * fro or n1 == 0.0:
            continue
        project(w)
        n2 = norm(w)
        if n2 == 0.0:
            continue
        be.set_column(Q, kept, w, 1.0 / n2)
        kept += 1
    return Q[:, :kept]


@dataclass
class DistResult:
    Q: object        # local rows of the basis
    U: object        # local rows of U
    sigma: object    # replicated
    V: object        # replicated
    est: float | None
    passes: int


def dist_randomized_svd(A_local, n, k, p, q, seed, comm, be, amax=None, estimate=True,
                        probes=config.DEFAULT_PROBES, alpha=config.DEFAULT_ALPHA,
                        truncate=False, sketch="gauss", speculative=True):
    """Alg 4.4 (q > 0) / 4.1 (q = 0) / 4.5 (sketch="srft") + Alg 5.1 +
    posterior estimate (reference rangefinder.py:49-82,221-265;
    factor.py:154-165; composition of cli.py:128-173,222-262) with A split by
    rows over `comm`.  Every rank returns its rows of Q and U and the
    replicated sigma, V and estimate.  `amax` is the global max|A| (fp32 /
    complex64 pass scaling).

    speculative: run the step without host synchronization (device-side
    decisions, one status all-reduce at the end) and fall back to the exact
    synchronous path on every rank if any rank flagged a rank drop or an
    unresolved pivot -- the single-GPU randomized_svd strategy."""
    ell = int(k) + int(p)
    if ell < 1 or ell > n:
        raise ValueError(f"rank+oversample {ell} must be in [1, {n}]")
    if sketch not in ("srft", "gauss", "gaussian"):
        raise ValueError(f"unknown sketch {sketch!r}")
    if sketch == "srft":
        if q > 0:
            raise ValueError("power iterations are not available with structured sketches")
        if not A_local.is_complex():
            raise NotImplementedError("row-sharded SRFT needs a complex A")
    args = (A_local, n, k, p, q, seed, comm, be, amax, estimate, probes, alpha, truncate, sketch)
    if speculative and hasattr(be, "chol_fast"):
        status = be.new_status(A_local)
        res = _dist_step(*args, status=status)
        flag = comm.allreduce_max(status.to(dtype=_float_of(status)))
        if be.status_value(flag) == 0:
            return res
    return _dist_step(*args, status=None)


def _float_of(t):
    import torch
    return torch.float64


def _dist_step(A_local, n, k, p, q, seed, comm, be, amax, estimate, probes, alpha, truncate,
               sketch, status):
    import contextlib
    ell = int(k) + int(p)
    spec = be.speculate(status) if status is not None else contextlib.nullcontext()

    def orth_m(Y):
        return dist_orth_fast(Y, comm, be, status) if status is not None else \
            dist_orth(Y, comm, be)

    with spec:
        if sketch == "srft":
            # the SRFT acts on the columns of A: every row block is sketched locally
            Q = orth_m(be.srft(A_local, ell, seed))
        else:
            Om = be.gaussian(n, ell, seed, _STREAM_GAUSS, A_local)
            Q = orth_m(be.pass_n(A_local, Om, amax))
        for _ in range(q):
            if Q.shape[1] == 0:
                break
            Z = comm.allreduce(be.pass_t(A_local, Q, amax))          # n x ell, replicated
            Qt = _replicated_orth(Z, be)
            Q = orth_m(be.pass_n(A_local, Qt, amax))
        if Q.shape[1] == 0:
            z = be.zeros_like_rows(A_local, 0)
            return DistResult(Q=Q, U=z, sigma=be.empty_sigma(A_local),
                              V=be.zeros_rows(n, 0, A_local), est=0.0,
                              passes=2 * q + 2 if q else 1)
        # Alg 5.1: Z = A^H Q (all-reduce), small SVD replicated, U_r = Q_r U~
        Z = comm.allreduce(be.pass_t(A_local, Q, amax))
        Ub, S, V = be.small_svd(Z)
        U = be.matmul(Q, Ub)
        est = None
        if estimate:
            W = be.gaussian(n, probes, seed + 13, _STREAM_PROBE, A_local)
            Zl = be.pass_n(A_local, W, amax)
            C = comm.allreduce(be.adj_matmul(Q, Zl))                 # Q^H Z, ell x r
            be.sub_(Zl, be.matmul(Q, C))
            ss = comm.allreduce(be.colsumsq(Zl))
            est = alpha * math.sqrt(2.0 / math.pi) * math.sqrt(be.to_scalar(ss))
    if truncate:
        kk = min(int(k), U.shape[1])
        U, S, V = U[:, :kk], S[:kk], V[:, :kk]
    return DistResult(Q=Q, U=U, sigma=S, V=V, est=est, passes=2 * q + 2 if q else 1)


def dist_randomized_svd_operator(op_local, n, k, p, q, seed, comm, be, estimate=True,
                                 probes=config.DEFAULT_PROBES, alpha=config.DEFAULT_ALPHA,
                                 truncate=False):
    """Row-sharded rSVD of an operator given by its row block A_r (m_r x n)
    on every rank -- the sparse path of config 5 (S_r + L_r R^T as a
    CudaCsrOperator over the rank's rows): Alg 4.4 / 4.1 +
    Alg 5.1 + the posterior estimate, with BOTH sides of the panels sharded.

      Y_r = A_r X                       X (n x ell) all-gathered from n-shards
      Z_c = sum_r (A_r^H Y_r)[c rows]   reduce-scatter of the n x ell partials
      orth of either side               dist_orth (all-reduced Gram)
      B = Q* A = Z^H:  Z = Q_Z R_Z (sharded CholeskyQR), SVD of R_Z^H replicated,
                       V_c = Q_Z,c W, U_r = Q_r U~

    so the n-side work is split too (the dense path replicates it: n = 4096
    there, n = 2^21 here).  Every rank returns its rows of Q and U, its
    n-side rows of V (row_range(n, rank, world)), sigma and the estimate."""
    ell = int(k) + int(p)
    if ell < 1 or ell > n:
        raise ValueError(f"rank+oversample {ell} must be in [1, {n}]")
    like = be.like(op_local)
    Om = be.gaussian(n, ell, seed, _STREAM_GAUSS, like)
    Q = dist_orth(be.op_n(op_local, Om), comm, be)
    for _ in range(q):
        if Q.shape[1] == 0:
            break
        Zc = comm.reduce_scatter_rows(be.op_t(op_local, Q), n)
        Qt = dist_orth(Zc, comm, be)
        X = comm.allgather_rows(Qt, n)
        Q = dist_orth(be.op_n(op_local, X), comm, be)
    passes = 2 * q + 2 if q else 1
    if Q.shape[1] == 0:
        return DistResult(Q=Q, U=be.zeros_like_rows(Q, 0), sigma=be.empty_sigma(like),
                          V=be.zeros_rows(row_range(n, comm.rank, comm.world)[1]
                                          - row_range(n, comm.rank, comm.world)[0], 0, like),
                          est=0.0, passes=passes)
    Zc = comm.reduce_scatter_rows(be.op_t(op_local, Q), n)
    QZ = dist_orth(Zc, comm, be, tol=0.0)
    if QZ.shape[1] == Q.shape[1]:
        RZ = comm.allreduce(be.adj_matmul(QZ, Zc))      # Z = Q_Z R_Z
        Ub, S, W = be.small_svd(RZ)                      # R_Z^H = Ub S W^H
        V = be.matmul(QZ, W)
    else:
        # numerically rank-deficient B: gather Z and factor it whole
        Ub, S, Vf = be.small_svd(comm.allgather_rows(Zc, n))
        a, b = row_range(n, comm.rank, comm.world)
        V = Vf[a:b]
    U = be.matmul(Q, Ub)
    est = None
    if estimate:
        W = be.gaussian(n, probes, seed + 13, _STREAM_PROBE, like)
        Zl = be.op_n(op_local, W)
        C = comm.allreduce(be.adj_matmul(Q, Zl))
        be.sub_(Zl, be.matmul(Q, C))
        ss = comm.allreduce(be.colsumsq(Zl))
        est = alpha * math.sqrt(2.0 / math.pi) * math.sqrt(be.to_scalar(ss))
    if truncate:
        kk = min(int(k), U.shape[1])
        U, S, V = U[:, :kk], S[:kk], V[:, :kk]
    return DistResult(Q=Q, U=U, sigma=S, V=V, est=est, passes=passes)


def row_range(m, rank, world):
    """Even row split [r0, r1) of m rows for `rank` of `world` (the cfg4
    recipe: rows split evenly over 1/2/4/8 GPUs)."""
    return m * rank // world, m * (rank + 1) // world


def sharded_randomized_svd(A_rows, k, p=config.DEFAULT_OVERSAMPLE, q=0, seed=0, sketch="gauss",
                           probes=config.DEFAULT_PROBES, alpha=config.DEFAULT_ALPHA,
                           estimate=True, truncate=False, group=None, device=None):
    """Public entry of the row-sharded path: each rank passes ITS rows of A
    (numpy / torch host or device array, same column count on every rank).
    Host inputs are copied to the rank's GPU and host outputs returned.
    Returns (U_rows, sigma, V, est) -- the same factors as randomized_svd
    (factor.py) on the stacked matrix."""
    import torch
    from .core import DenseOperator, is_device_array, to_hosts
    host = not is_device_array(A_rows)
    comm = Comm(group)
    # upload, finiteness check and local max|A|; the verdict is agreed on by
    # all ranks so that a bad shard raises everywhere instead of hanging peers
    err = None
    try:
        op = DenseOperator(A_rows, device=device)
    except ValueError as e:
        err = e
    dev = torch.cuda.current_device() if device is None else device
    flag = torch.tensor([0.0 if err is None else 1.0], dtype=torch.float64, device=f"cuda:{dev}")
    if float(comm.allreduce_max(flag).item()) != 0.0:
        raise err if err is not None else ValueError("matrix shard on another rank is invalid")
    A = op.array
    amax = None
    if A.dtype in (torch.float32, torch.complex64):
        t = torch.tensor([float(op.amax)], dtype=torch.float64, device=A.device)
        amax = float(comm.allreduce_max(t).item())
    res = dist_randomized_svd(A, A.shape[1], k, p, q, seed, comm, GpuBackend(), amax=amax,
                              estimate=estimate, probes=probes, alpha=alpha, truncate=truncate,
                              sketch=sketch)
    if host:
        return (*to_hosts(res.U, res.sigma, res.V), res.est)
    return res.U, res.sigma, res.V, res.est


def _replicated_orth(Z, be):
    """Orthonormalization of a replicated n x ell panel (every rank computes
    the same Q~ from the same Z)."""
    if hasattr(be, "orth_local"):
        return be.orth_local(Z)
    from .core import orth_dev
    return orth_dev(Z)
