"""numpy restatement of the reference's randomized-SVD hot path (CPU oracle).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  This module is the
checker the CUDA path is compared against, and the CPU reference arm that
bench.py times.  It restates the algorithms of the reference package
``lowrank`` (``/root/reference/pkg/src/lowrank``) function by function; each
function names the reference file:line it follows.  The reference is not
imported here (it does not exist on the GPU box); instead tests/golden holds
vectors produced by the reference itself (tests/golden/make_golden.py) and
tests/test_oracle_golden.py pins this restatement to them.

Arithmetic matches the reference: everything is promoted to float64 /
complex128 (reference core.py:44-47, sketch.py:189), matrix products go
through numpy/OpenBLAS, the small SVD through LAPACK gesdd.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# reference config.py:9,19,22-23
GS_DROP_TOL = 1e-10
DEFAULT_OVERSAMPLE = 5
DEFAULT_PROBES = 10
DEFAULT_ALPHA = 10.0

# Philox stream tags, reference sketch.py:26-29 and rangefinder.py:78
STREAM_GAUSS = 0x67617573      # "gaus"
STREAM_SRFT = 0x73726674       # "srft"
STREAM_GSRFT = 0x67737266      # "gsrf"  (sketch.py:28)
STREAM_PROBE = 0x70726F62      # "prob"
STREAM_SYNTH = 0x73796E74      # "synt"  (oracle.py:120)


# ---------------------------------------------------------------------------
# Random draws (host side; the CUDA path uploads the same arrays)

def rng_for(seed, stream=0, index=0):
    """Philox generator keyed by seed | stream<<64 | index<<96.

    Follows reference sketch.py:32-42: the 128-bit Philox key packs the
    64-bit seed, a 32-bit stream tag and a 32-bit draw index.
    """
    key = int(seed) % (1 << 64)
    key |= (int(stream) % (1 << 32)) << 64
    key |= (int(index) % (1 << 32)) << 96
    return np.random.Generator(np.random.Philox(key=key))


def gaussian_matrix(n, ell, seed):
    """n x ell standard normals, row-major draw order (sketch.py:96-100)."""
    if n < 1 or ell < 1:
        raise ValueError("dimensions must be >= 1")
    return rng_for(seed, STREAM_GAUSS).standard_normal((n, ell))


def probe_matrix(n, r, seed):
    """Estimator probes W (rangefinder.py:78)."""
    return rng_for(seed, STREAM_PROBE).standard_normal((n, r))


@dataclass
class SrftDraw:
    """Materialized SRFT test matrix scale * diag(d) F R (sketch.py:207-218)."""

    n: int
    ell: int
    d: np.ndarray
    picks: np.ndarray
    scale: float


def srft_operator(n, ell, seed):
    """d = exp(2 pi i U[0,1)), then picks = permutation(n)[:ell] from the
    same stream (sketch.py:246-256)."""
    if ell > n:
        raise ValueError("sample count exceeds dimension")
    g = rng_for(seed, STREAM_SRFT)
    d = np.exp(2j * np.pi * g.random(n))
    picks = g.permutation(n)[:ell]
    return SrftDraw(n=n, ell=ell, d=d, picks=picks, scale=float(np.sqrt(n / ell)))


# ---------------------------------------------------------------------------
# FFT (reference sketch.py:115-200): radix-2 for powers of two, chirp-z
# (Bluestein) otherwise, unitary scaling n^-1/2.

def _bit_reversal(n):
    bits = n.bit_length() - 1
    idx = np.arange(n)
    rev = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        rev |= ((idx >> b) & 1) << (bits - 1 - b)
    return rev


def fft_radix2(X, inverse=False):
    """Unnormalized iterative radix-2 DIT FFT along the last axis
    (sketch.py:129-148): bit-reverse, then log2(n) butterfly stages."""
    n = X.shape[-1]
    Y = np.ascontiguousarray(X[..., _bit_reversal(n)], dtype=np.complex128)
    sgn = 1.0 if inverse else -1.0
    span = 2
    while span <= n:
        h = span // 2
        tw = np.exp(sgn * 2j * np.pi * np.arange(h) / span)
        view = Y.reshape(Y.shape[:-1] + (n // span, span))
        top = view[..., :h]
        bot = view[..., h:] * tw
        lo = top - bot
        view[..., :h] = top + bot
        view[..., h:] = lo
        span *= 2
    return Y


def fft_bluestein(X, inverse=False):
    """Arbitrary-length DFT by chirp convolution (sketch.py:155-176)."""
    n = X.shape[-1]
    sgn = 1.0 if inverse else -1.0
    t = np.arange(n, dtype=np.int64)
    w = np.exp(sgn * 1j * np.pi * ((t * t) % (2 * n)) / n)
    L = 1 << (2 * n - 2).bit_length()
    a = np.zeros(X.shape[:-1] + (L,), dtype=np.complex128)
    a[..., :n] = X * w
    b = np.zeros(L, dtype=np.complex128)
    b[:n] = np.conj(w)
    b[L - n + 1:] = np.conj(w[1:][::-1])
    conv = fft_radix2(fft_radix2(a) * fft_radix2(b[None, :])[0], inverse=True) / L
    return conv[..., :n] * w


def dft(v, axis=-1):
    """Unitary DFT, f_pq = n^-1/2 exp(-2 pi i pq / n) (sketch.py:179-200)."""
    v = np.asarray(v)
    if v.ndim == 0:
        raise ValueError("dft expects a vector or matrix")
    X = np.moveaxis(v, axis, -1).astype(np.complex128)
    n = X.shape[-1]
    if n == 1:
        out = X.copy()
    elif n & (n - 1) == 0:
        out = fft_radix2(X)
    else:
        out = fft_bluestein(X)
    return np.moveaxis(out / np.sqrt(n), -1, axis)


def srft_apply(A, draw):
    """Y = scale * dft(A * d)[:, picks] (sketch.py:306-320)."""
    A = np.asarray(A)
    if draw.n != A.shape[1]:
        raise ValueError("operator dimension does not match matrix columns")
    return dft(A * draw.d[None, :], axis=1)[:, draw.picks] * draw.scale


@dataclass
class GsrftDraw:
    """Givens-chain SRFT draw (sketch.py:221-243): x -> x D'' Theta' D' Theta D F R."""
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


def gsrft_operator(n, ell, seed):
    """Draw order of sketch.py:259-275: d_outer, perm_outer, thetas_outer,
    d_mid, perm_inner, thetas_inner, d_inner, picks -- one stream."""
    if ell > n:
        raise ValueError("sample count exceeds dimension")
    g = rng_for(seed, STREAM_GSRFT)
    d_outer = np.exp(2j * np.pi * g.random(n))
    perm_outer = g.permutation(n)
    thetas_outer = g.uniform(0.0, 2.0 * np.pi, max(n - 1, 0))
    d_mid = np.exp(2j * np.pi * g.random(n))
    perm_inner = g.permutation(n)
    thetas_inner = g.uniform(0.0, 2.0 * np.pi, max(n - 1, 0))
    d_inner = np.exp(2j * np.pi * g.random(n))
    picks = g.permutation(n)[:ell]
    return GsrftDraw(n, ell, d_outer, perm_outer, thetas_outer, d_mid, perm_inner,
                     thetas_inner, d_inner, picks, float(np.sqrt(n / ell)))


def givens_chain(X, perm, thetas):
    """X[:, perm] then the ascending plane rotations on column pairs
    (i, i+1): [a, b] <- [c a - s b, s a + c b]  (sketch.py:278-291)."""
    Y = X[:, perm].astype(np.complex128, copy=True)
    c, s = np.cos(thetas), np.sin(thetas)
    for i in range(len(thetas)):
        a = Y[:, i].copy()
        b = Y[:, i + 1].copy()
        Y[:, i] = c[i] * a - s[i] * b
        Y[:, i + 1] = s[i] * a + c[i] * b
    return Y


def gsrft_apply(A, draw):
    """Y = A Omega for the Givens-chain SRFT (sketch.py:323-337)."""
    A = np.asarray(A)
    if draw.n != A.shape[1]:
        raise ValueError("operator dimension does not match matrix columns")
    Y = A * draw.d_outer[None, :]
    Y = givens_chain(Y, draw.perm_outer, draw.thetas_outer)
    Y = Y * draw.d_mid[None, :]
    Y = givens_chain(Y, draw.perm_inner, draw.thetas_inner)
    Y = Y * draw.d_inner[None, :]
    return dft(Y, axis=1)[:, draw.picks] * draw.scale


# ---------------------------------------------------------------------------
# Dense kernels (reference core.py)

def as_matrix(a):
    """2-D, nonempty, finite; promoted to float64/complex128 (core.py:33-50)."""
    arr = np.asarray(a)
    if arr.ndim != 2:
        raise ValueError(f"matrix must be 2-D, got shape {arr.shape}")
    if arr.size == 0:
        raise ValueError("matrix must be nonempty")
    arr = arr.astype(np.complex128 if np.iscomplexobj(arr) else np.float64, copy=False)
    if not np.all(np.isfinite(arr)):
        raise ValueError("matrix contains non-finite entries")
    return arr


def orthonormalize_double_gs(Y, tol=GS_DROP_TOL):
    """Column-wise classical Gram-Schmidt with one reorthogonalization
    (core.py:84-115).  Column j is dropped when its residual after the first
    projection is <= tol * ||Y||_F (or exactly zero), or when the residual
    after the second projection is exactly zero.  Accepted columns are kept
    in a Fortran-ordered buffer instead of being re-stacked every step; the
    arithmetic per column is the reference's w - Q (Q* w), twice."""
    Y = np.asarray(Y)
    m, ell = Y.shape
    cplx = np.iscomplexobj(Y)
    dt = np.complex128 if cplx else np.float64
    fro = np.linalg.norm(Y)
    buf = np.zeros((m, ell), dtype=dt, order="F")
    kept = 0
    for j in range(ell):
        w = Y[:, j].astype(dt)
        Q = buf[:, :kept]
        if kept:
            w = w - Q @ (Q.conj().T @ w)
        nrm = np.linalg.norm(w)
        if nrm <= tol * fro or nrm == 0.0:
            continue
        if kept:
            w = w - Q @ (Q.conj().T @ w)
        nrm = np.linalg.norm(w)
        if nrm == 0.0:
            continue
        buf[:, kept] = w / nrm
        kept += 1
    if kept == 0:
        return np.zeros((m, 0), dtype=Y.dtype)
    return np.ascontiguousarray(buf[:, :kept])


def plain_gs(Y):
    """Unsafeguarded single-pass CGS, no drops (rangefinder.py:169-184)."""
    Q = np.array(Y, dtype=np.complex128 if np.iscomplexobj(Y) else np.float64)
    for j in range(Q.shape[1]):
        for i in range(j):
            Q[:, j] -= Q[:, i] * np.vdot(Q[:, i], Q[:, j])
        nrm = np.linalg.norm(Q[:, j])
        if nrm > 0:
            Q[:, j] /= nrm
    return Q


@dataclass
class SmallSVD:
    U: np.ndarray
    sigma: np.ndarray
    V: np.ndarray


def sign_fix(U, V):
    """Rotate the first entry of each left vector with |u| > 1e-10 max|u|
    onto the positive real axis; V absorbs the same phase (core.py:221-229)."""
    for j in range(U.shape[1]):
        mag = np.abs(U[:, j])
        top = mag.max() if mag.size else 0.0
        idx = np.flatnonzero(mag > 1e-10 * top)
        if idx.size == 0:
            continue
        z = U[idx[0], j]
        ph = z / abs(z)
        U[:, j] *= np.conj(ph)
        V[:, j] *= np.conj(ph)
    return U, V


def small_svd(B):
    """Thin SVD by LAPACK gesdd, gesvd retry (core.py:199-230)."""
    B = np.asarray(B)
    try:
        U, s, Vh = np.linalg.svd(B, full_matrices=False)
    except np.linalg.LinAlgError:
        import scipy.linalg
        U, s, Vh = scipy.linalg.svd(B, full_matrices=False, lapack_driver="gesvd")
    V = Vh.conj().T
    U, V = sign_fix(U, V)
    return SmallSVD(U=U, sigma=s.astype(np.float64), V=V)


# ---------------------------------------------------------------------------
# Operators (core.py:332-402)

@dataclass
class Counters:
    matvecs: int = 0
    adjoint_matvecs: int = 0
    passes: int = 0
    flops: int = 0


class Operator:
    """Counting m x n operator: apply / apply_adjoint add cols matvecs, one
    pass and 2*m*n*cols flops each (core.py:360-374)."""

    def __init__(self, m, n):
        self.m, self.n = int(m), int(n)
        self.counters = Counters()

    @property
    def shape(self):
        return (self.m, self.n)

    def _count(self, X, adjoint):
        cols = 1 if np.ndim(X) == 1 else np.shape(X)[1]
        if adjoint:
            self.counters.adjoint_matvecs += cols
        else:
            self.counters.matvecs += cols
        self.counters.passes += 1
        self.counters.flops += 2 * self.m * self.n * cols

    def apply(self, X):
        self._count(X, False)
        return self._apply(np.asarray(X))

    def apply_adjoint(self, Y):
        self._count(Y, True)
        return self._apply_adjoint(np.asarray(Y))


class Dense(Operator):
    """In-memory dense A (core.py:383-395), promoted by as_matrix."""

    def __init__(self, A, promote=True):
        A = as_matrix(A) if promote else np.asarray(A)
        super().__init__(*A.shape)
        self.array = A

    def _apply(self, X):
        return self.array @ X

    def _apply_adjoint(self, Y):
        return self.array.conj().T @ Y


class Blockwise(Operator):
    """Row-block fp64 application of a lower-precision stored A.

    Arithmetic-identical to Dense(A) (each block is promoted to float64 and
    multiplied) without holding an fp64 copy of all of A; the row-block
    structure follows the reference's RowBlockStream (io.py:319-388).  Used
    for the config-4 CPU baseline, whose fp64 upcast would not fit in host
    RAM."""

    def __init__(self, A, block_rows=65536):
        super().__init__(*A.shape)
        self.array = A
        self.block = int(block_rows)

    def _apply(self, X):
        X = np.asarray(X, dtype=np.float64)
        out = np.empty((self.m,) + X.shape[1:], dtype=np.float64)
        for r in range(0, self.m, self.block):
            out[r:r + self.block] = self.array[r:r + self.block].astype(np.float64) @ X
        return out

    def _apply_adjoint(self, Y):
        Y = np.asarray(Y, dtype=np.float64)
        acc = np.zeros((self.n,) + Y.shape[1:], dtype=np.float64)
        for r in range(0, self.m, self.block):
            acc += self.array[r:r + self.block].astype(np.float64).T @ Y[r:r + self.block]
        return acc


class SparsePlusLowRank(Operator):
    """S + L R^T with S in scipy CSR (config 5; no reference code exists for
    sparse A -- SURVEY.md §8c "parity unpinned" -- so this is the user
    MatVecOperator subclass the survey prescribes)."""

    def __init__(self, S, L, R):
        super().__init__(*S.shape)
        self.S, self.L, self.R = S, np.asarray(L), np.asarray(R)
        self.St = S.T.tocsr()

    def _apply(self, X):
        return self.S @ X + self.L @ (self.R.T @ X)

    def _apply_adjoint(self, Y):
        return self.St @ Y + self.R @ (self.L.T @ Y)


def as_operator(A):
    return A if isinstance(A, Operator) else Dense(A)


# ---------------------------------------------------------------------------
# Stage A (rangefinder.py)

@dataclass
class RangeBasis:
    Q: np.ndarray
    samples_used: int
    passes: int
    est_error: float | None
    kind: str = "gaussian"
    ell: int = 1
    power_q: int = 0
    seed: int = 0
    diagnostics: dict = field(default_factory=dict)
    saturated: bool = False
    probe_matvecs: int = 0


def _check_ell(op, ell):
    if not 1 <= ell <= min(op.shape):
        raise ValueError("ell must satisfy 1 <= ell <= min(m, n)")


def randomized_range_finder(A, ell, seed, ortho_tol=GS_DROP_TOL):
    """Alg 4.1 (rangefinder.py:49-62): Q = DGS(A Omega), one pass."""
    op = as_operator(A)
    _check_ell(op, ell)
    Q = orthonormalize_double_gs(op.apply(gaussian_matrix(op.n, ell, seed)), tol=ortho_tol)
    return RangeBasis(Q=Q, samples_used=ell, passes=1,
                      est_error=0.0 if Q.shape[1] == 0 else None, ell=ell, seed=seed)


def power_iteration_range(A, ell, q, seed, ortho_tol=GS_DROP_TOL, safeguarded=True):
    """Alg 4.3 (rangefinder.py:187-218): orthonormalize (A A*)^q A Omega."""
    if q < 0:
        raise ValueError("q must be nonnegative")
    op = as_operator(A)
    _check_ell(op, ell)
    Y = op.apply(gaussian_matrix(op.n, ell, seed))
    for _ in range(q):
        Y = op.apply(op.apply_adjoint(Y))
    Q = orthonormalize_double_gs(Y, tol=ortho_tol) if safeguarded else plain_gs(Y)
    return RangeBasis(Q=Q, samples_used=ell, passes=2 * q + 2,
                      est_error=0.0 if Q.shape[1] == 0 else None, ell=ell,
                      power_q=q, seed=seed)


def subspace_iteration_range(A, ell, q, seed, ortho_tol=GS_DROP_TOL):
    """Alg 4.4 (rangefinder.py:221-243): re-orthonormalize after every
    application of A and A*."""
    if q < 0:
        raise ValueError("q must be nonnegative")
    op = as_operator(A)
    _check_ell(op, ell)
    Q = orthonormalize_double_gs(op.apply(gaussian_matrix(op.n, ell, seed)), tol=ortho_tol)
    for _ in range(q):
        Qt = orthonormalize_double_gs(op.apply_adjoint(Q), tol=ortho_tol)
        Q = orthonormalize_double_gs(op.apply(Qt), tol=ortho_tol)
    return RangeBasis(Q=Q, samples_used=ell, passes=2 * q + 2,
                      est_error=0.0 if Q.shape[1] == 0 else None, ell=ell,
                      power_q=q, seed=seed)


STREAM_ADAPT = 0x61646170      # "adap" (rangefinder.py:121)


def adaptive_range_finder(A, eps, r=DEFAULT_PROBES, seed=0, alpha=DEFAULT_ALPHA, block=1):
    """Alg 4.2 (rangefinder.py:89-159): grow the basis one vector at a time
    from probe residuals y = (I - QQ*) A w; batch b of `block` probes is
    drawn from Philox(seed, "adap", index = draws so far); stop once the r
    oldest pending residual norms are <= eps / (alpha sqrt(2/pi))."""
    if eps <= 0:
        raise ValueError("eps must be positive")
    if r < 1:
        raise ValueError("r must be >= 1")
    block = max(int(block), 1)
    op = as_operator(A)
    m, n = op.shape
    threshold = eps / (alpha * math.sqrt(2.0 / math.pi))
    draws = 0
    pending, cols = [], []
    saturated = False
    while True:
        while len(pending) < r:
            W = rng_for(seed, STREAM_ADAPT, draws).standard_normal((n, block))
            draws += block
            fresh = op.apply(W)
            if cols:
                Qc = np.column_stack(cols)
                fresh = fresh - Qc @ (Qc.conj().T @ fresh)
            pending.extend(fresh[:, i] for i in range(fresh.shape[1]))
        if max(np.linalg.norm(y) for y in pending[:r]) <= threshold:
            break
        y = pending.pop(0)
        Q = np.column_stack(cols) if cols else np.zeros((m, 0))
        y = y - Q @ (Q.conj().T @ y)
        nrm = np.linalg.norm(y)
        if nrm == 0.0:
            continue
        q = y / nrm
        cols.append(q)
        if len(cols) >= min(m, n):
            saturated = True
            break
        for i in range(len(pending)):
            pending[i] = pending[i] - q * np.vdot(q, pending[i])
    Q = np.column_stack(cols) if cols else np.zeros((m, 0))
    est = (alpha * math.sqrt(2.0 / math.pi) * max(np.linalg.norm(y) for y in pending[:r])
           if pending else 0.0)
    return RangeBasis(Q=Q, samples_used=draws, passes=1, est_error=float(est), kind="gaussian",
                      ell=1, seed=seed, saturated=saturated, probe_matvecs=r)


def fast_range_finder(A, ell, seed, ortho_tol=GS_DROP_TOL, kind="srft"):
    """Alg 4.5 with the SRFT or its Givens-chain variant (rangefinder.py:246-266)."""
    A = np.asarray(A)
    if kind not in ("srft", "gsrft"):
        raise ValueError("kind must be 'srft' or 'gsrft'")
    if kind == "srft":
        Y = srft_apply(A, srft_operator(A.shape[1], ell, seed))
    else:
        Y = gsrft_apply(A, gsrft_operator(A.shape[1], ell, seed))
    diag = {}
    if not np.iscomplexobj(A):
        diag["max_imag_sample"] = float(np.abs(Y.imag).max())
    Q = orthonormalize_double_gs(Y, tol=ortho_tol)
    return RangeBasis(Q=Q, samples_used=ell, passes=1,
                      est_error=0.0 if Q.shape[1] == 0 else None, kind=kind,
                      ell=ell, seed=seed, diagnostics=diag)


def posterior_error_estimate(A, Q, r=DEFAULT_PROBES, alpha=DEFAULT_ALPHA, seed=0):
    """alpha sqrt(2/pi) max_i ||(I - QQ*) A w_i|| (rangefinder.py:65-82)."""
    if r < 1:
        raise ValueError("r must be >= 1")
    if alpha <= 1:
        raise ValueError("alpha must exceed 1")
    op = as_operator(A)
    Z = op.apply(probe_matrix(op.n, r, seed))
    if Q.shape[1]:
        Z = Z - Q @ (Q.conj().T @ Z)
    return float(alpha * math.sqrt(2.0 / math.pi) * np.linalg.norm(Z, axis=0).max())


# ---------------------------------------------------------------------------
# Stage B (factor.py)

@dataclass
class PartialSVD:
    U: np.ndarray
    sigma: np.ndarray
    V: np.ndarray

    def compose(self):
        return (self.U * self.sigma) @ self.V.conj().T


def direct_svd(A, Q):
    """Alg 5.1 (factor.py:154-165): B = (A* Q)*, small SVD, U = Q U~."""
    op = as_operator(A)
    if Q.shape[0] != op.m:
        raise ValueError("basis rows must match matrix rows")
    f = small_svd(op.apply_adjoint(Q).conj().T)
    return PartialSVD(U=Q @ f.U, sigma=f.sigma, V=f.V)


def truncate_rank(f, k):
    """Top-k slice (factor.py:408-426, PartialSVD branch)."""
    if k > len(f.sigma):
        raise ValueError("k exceeds current rank")
    return PartialSVD(U=f.U[:, :k], sigma=f.sigma[:k], V=f.V[:, :k])


# ---------------------------------------------------------------------------
# Hermitian Stage-B routes (reference factor.py:168-191,300-335, core.py:233-294)

PSD_TOL = 1e-12                 # reference config.py:16
TRIANGULAR_TRUNC_TOL = 1e-12    # reference config.py:12


class NotPSDError(ValueError):
    """reference core.py:29-30"""


def small_eig_hermitian(B):
    """Symmetrize, LAPACK eigh, order by descending |lam| then descending lam
    (core.py:233-246)."""
    B = np.asarray(B)
    H = 0.5 * (B + B.conj().T)
    lam, V = np.linalg.eigh(H)
    order = np.lexsort((-lam, -np.abs(lam)))
    return V[:, order], lam[order].astype(np.float64)


def cholesky_psd(B, tol=PSD_TOL):
    """Upper C with B = C* C; pivots in [-tol ||B||_2, 0] clamp to zero, below
    raise NotPSDError (core.py:249-272)."""
    B = np.asarray(B)
    n = B.shape[0]
    scale = np.linalg.norm(B, 2) if n else 0.0
    C = np.zeros_like(B, dtype=np.complex128 if np.iscomplexobj(B) else np.float64)
    for i in range(n):
        d = B[i, i].real - np.real(C[:i, i].conj() @ C[:i, i])
        if d < -tol * scale:
            raise NotPSDError(f"matrix is not PSD: pivot {d:.3e} at index {i}")
        d = max(d, 0.0)
        C[i, i] = np.sqrt(d)
        if i + 1 < n:
            if C[i, i] > 0:
                C[i, i + 1:] = (B[i, i + 1:] - C[:i, i].conj() @ C[:i, i + 1:]) / C[i, i]
            else:
                C[i, i + 1:] = 0.0
    return C


def solve_triangular_trunc(R, B, trunc_tol=TRIANGULAR_TRUNC_TOL):
    """Back substitution with zero components for diagonals <= trunc_tol
    |r|_max (core.py:275-294)."""
    R = np.asarray(R)
    B = np.asarray(B)
    k = R.shape[0]
    X = np.zeros((k,) + B.shape[1:], dtype=np.promote_types(R.dtype, B.dtype))
    diag = np.abs(np.diagonal(R))
    cutoff = trunc_tol * (diag.max() if k else 0.0)
    for i in range(k - 1, -1, -1):
        if diag[i] <= cutoff:
            continue
        X[i] = (B[i] - R[i, i + 1:] @ X[i + 1:]) / R[i, i]
    return X


@dataclass
class PartialEig:
    U: np.ndarray
    lam: np.ndarray
    diagnostics: dict = field(default_factory=dict)

    def compose(self):
        return (self.U * self.lam) @ self.U.conj().T


def hermitian_probe(op, seed=0, tol=1e-8):
    """factor.py:168-178 (numpy default_rng draws, two applications)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(op.n)
    y = rng.standard_normal(op.n)
    ax = op.apply(x)
    ay = op.apply(y)
    lhs, rhs = np.vdot(y, ax), np.vdot(ay, x)
    denom = max(abs(lhs), abs(rhs), 1e-300)
    if abs(lhs - rhs) / denom > tol:
        raise ValueError("operator failed the Hermitian probe")


def direct_eig_hermitian(A, Q):
    """factor.py:181-191: B = Q* A Q, eigenpairs of B, U = Q V."""
    op = as_operator(A)
    hermitian_probe(op)
    B = Q.conj().T @ op.apply(Q)
    V, lam = small_eig_hermitian(B)
    return PartialEig(U=Q @ V, lam=lam)


def eig_nystrom(A, Q):
    """factor.py:300-335: F = (AQ) C^{-1} with B2 = Q*AQ = C*C (PSD
    Cholesky), eigen fallback with clamping when B2 is not PSD; lam =
    sigma(F)^2.  Returns (PartialEig, F)."""
    op = as_operator(A)
    B1 = op.apply(Q)
    B2 = Q.conj().T @ B1
    B2 = 0.5 * (B2 + B2.conj().T)
    diagnostics = {}
    try:
        C = cholesky_psd(B2)
        Ft = solve_triangular_trunc(C.conj().T[::-1, ::-1], B1.conj().T[::-1])[::-1]
        F = Ft.conj().T
    except NotPSDError as exc:
        V, lam = small_eig_hermitian(B2)
        diagnostics["not_psd_fallback"] = True
        diagnostics["min_projected_eigenvalue"] = float(lam.min())
        diagnostics["detail"] = str(exc)
        lam_c = np.clip(lam, 0.0, None)
        inv_root = np.where(lam_c > 1e-15 * max(lam_c.max(), 1e-300),
                            1.0 / np.sqrt(np.where(lam_c > 0, lam_c, 1.0)), 0.0)
        F = B1 @ (V * inv_root)
    f = small_svd(F)
    return PartialEig(U=f.U, lam=f.sigma ** 2, diagnostics=diagnostics), F


# ---------------------------------------------------------------------------
# Verification helpers (reference oracle.py)

def exact_projection_error(A, Q, norm="spectral"):
    """||(I - QQ*) A|| by explicit residual (oracle.py:25-40)."""
    A = np.asarray(A)
    R = A - Q @ (Q.conj().T @ A) if Q.shape[1] else A
    if norm == "spectral":
        return float(np.linalg.svd(R, compute_uv=False)[0]) if min(R.shape) else 0.0
    return float(np.linalg.norm(R))


def principal_angles(Q1, Q2):
    """Principal angles between two orthonormal bases."""
    s = np.linalg.svd(Q1.conj().T @ Q2, compute_uv=False)
    return np.arccos(np.clip(s, -1.0, 1.0))


def jacobi_singular_values(A, sweeps=60, tol=1e-15):
    """One-sided cyclic Jacobi singular values -- an SVD cross-check that does
    not share LAPACK's code path (cf. reference oracle.py:230-267)."""
    M = np.array(A, dtype=np.float64)
    if M.shape[0] < M.shape[1]:
        M = M.T.copy()
    n = M.shape[1]
    for _ in range(sweeps):
        off = 0.0
        for p in range(n - 1):
            for q in range(p + 1, n):
                a = M[:, p] @ M[:, p]
                b = M[:, q] @ M[:, q]
                c = M[:, p] @ M[:, q]
                if abs(c) <= tol * math.sqrt(a * b) or c == 0.0:
                    continue
                off = max(off, abs(c) / math.sqrt(a * b))
                zeta = (b - a) / (2.0 * c)
                t = math.copysign(1.0, zeta) / (abs(zeta) + math.sqrt(1.0 + zeta * zeta))
                cs = 1.0 / math.sqrt(1.0 + t * t)
                sn = cs * t
                mp = M[:, p].copy()
                M[:, p] = cs * mp - sn * M[:, q]
                M[:, q] = sn * mp + cs * M[:, q]
        if off <= tol:
            break
    return np.sort(np.linalg.norm(M, axis=0))[::-1]


def rsvd(A, k, p, q, seed, sketch="gauss", probes=DEFAULT_PROBES, alpha=DEFAULT_ALPHA,
         estimate=True):
    """The composition the reference CLI calls "randomized SVD"
    (cli.py:128-173 Stage-A dispatch, 222-262 _cmd_svd): ell = k + p;
    gauss q>0 -> Alg 4.4, gauss q=0 -> Alg 4.1, srft -> Alg 4.5; then
    direct_svd and the posterior estimate with seed + 13."""
    op = as_operator(A)
    ell = k + p
    if sketch == "gauss":
        basis = (subspace_iteration_range(op, ell, q, seed) if q > 0
                 else randomized_range_finder(op, ell, seed))
    else:
        if q > 0:
            raise ValueError("power iterations are not available with structured sketches")
        basis = fast_range_finder(op.array, ell, seed, kind=sketch)
    f = direct_svd(op, basis.Q)
    est = basis.est_error
    if est is None and estimate:
        est = posterior_error_estimate(op, basis.Q, r=probes, alpha=alpha, seed=seed + 13)
    return basis, f, est


# ---------------------------------------------------------------------------
# One-pass sketches and row-block streaming (reference factor.py:95-147,
# 338-401; io.py:35,178-204,319-430; core.py:133-186,297-325)

ONE_PASS_DIM_CAP = 250_000       # reference config.py:31
ONE_PASS_COND_WARN = 1e12        # reference config.py:34
LRK_MAGIC = b"LRKMAT00"          # reference io.py:35


def write_matrix_binary(A, path):
    """io.py:178-188."""
    A = as_matrix(A)
    with open(path, "wb") as fh:
        fh.write(LRK_MAGIC)
        np.asarray([1 if np.iscomplexobj(A) else 0, A.shape[0], A.shape[1]],
                   dtype="<i8").tofile(fh)
        np.ascontiguousarray(A).astype("<c16" if np.iscomplexobj(A) else "<f8").tofile(fh)


def stream_row_blocks(path, block_rows):
    """io.py:319-356: (row, block) pairs of a LRKMAT00 file."""
    with open(path, "rb") as fh:
        if fh.read(8) != LRK_MAGIC:
            raise ValueError(f"{path}: bad magic")
        code, m, n = (int(x) for x in np.fromfile(fh, dtype="<i8", count=3))
        dtype = "<c16" if code == 1 else "<f8"
        row = 0
        while row < m:
            rows = min(block_rows, m - row)
            data = np.fromfile(fh, dtype=dtype, count=rows * n)
            if data.size != rows * n:
                raise IOError(f"{path}: stream truncated at row block starting {row}")
            yield row, data.reshape(rows, n)
            row += rows


def accumulate_two_sided_samples(blocks, m, n, ell, ell_tilde, seed):
    """io.py:364-388."""
    Omega = gaussian_matrix(n, ell, seed)
    Omega_t = gaussian_matrix(m, ell_tilde, seed + 1)
    Y = Yt = None
    total = 0
    for row, block in blocks:
        if Y is None:
            dt = np.promote_types(block.dtype, Omega.dtype)
            Y = np.zeros((m, ell), dtype=dt)
            Yt = np.zeros((n, ell_tilde), dtype=dt)
        rows = block.shape[0]
        Y[row:row + rows, :] = block @ Omega
        Yt += block.conj().T @ Omega_t[row:row + rows, :]
        total += rows
    if total != m:
        raise IOError(f"stream delivered {total} rows, expected {m}")
    return Omega, Omega_t, Y, Yt


@dataclass
class SampleBundle:
    """factor.py:95-113."""
    Omega: np.ndarray
    Y: np.ndarray
    Q: np.ndarray
    Omega_tilde: np.ndarray = None
    Y_tilde: np.ndarray = None
    Q_tilde: np.ndarray = None
    q_choice: str = "gs"
    seed: int = None


def _basis_from_samples(Y, rank=None, ortho_tol=GS_DROP_TOL):
    """factor.py:116-120."""
    if rank is None:
        return orthonormalize_double_gs(Y, tol=ortho_tol), "gs"
    return small_svd(Y).U[:, :rank], "svd"


def sample_bundle(A, ell, seed, rank=None):
    """factor.py:123-133."""
    op = as_operator(A)
    Omega = gaussian_matrix(op.n, ell, seed)
    Y = op.apply(Omega)
    Q, choice = _basis_from_samples(Y, rank)
    return SampleBundle(Omega=Omega, Y=Y, Q=Q, q_choice=choice, seed=seed)


def sample_bundle_two_sided(A, ell, ell_tilde=None, seed=0, rank=None):
    """factor.py:136-147."""
    op = as_operator(A)
    ell_tilde = ell if ell_tilde is None else ell_tilde
    Omega = gaussian_matrix(op.n, ell, seed)
    Omega_t = gaussian_matrix(op.m, ell_tilde, seed + 1)
    Y = op.apply(Omega)
    Yt = op.apply_adjoint(Omega_t)
    Q, choice = _basis_from_samples(Y, rank)
    Qt, _ = _basis_from_samples(Yt, rank)
    return SampleBundle(Omega=Omega, Y=Y, Q=Q, Omega_tilde=Omega_t, Y_tilde=Yt, Q_tilde=Qt,
                        q_choice=choice, seed=seed)


def streamed_sample_bundle(path, block_rows, ell, ell_tilde=None, seed=0, rank=None):
    """io.py:391-404 over a file."""
    with open(path, "rb") as fh:
        fh.read(8)
        _, m, n = (int(x) for x in np.fromfile(fh, dtype="<i8", count=3))
    ell_tilde = ell if ell_tilde is None else ell_tilde
    Omega, Omega_t, Y, Yt = accumulate_two_sided_samples(stream_row_blocks(path, block_rows), m, n,
                                                         ell, ell_tilde, seed)
    Q, choice = _basis_from_samples(Y, rank)
    Qt, _ = _basis_from_samples(Yt, rank)
    return SampleBundle(Omega=Omega, Y=Y, Q=Q, Omega_tilde=Omega_t, Y_tilde=Yt, Q_tilde=Qt,
                        q_choice=choice, seed=seed)


def pivoted_qr_r(A):
    """Column-pivoted QR (core.py:133-186, Businger-Golub: largest remaining
    column norm, ties to the lowest index): (Q, R, perm) with A[:, perm] =
    Q R.  scipy's geqp3 makes the same greedy choice."""
    import scipy.linalg
    Q, R, perm = scipy.linalg.qr(np.asarray(A), mode="economic", pivoting=True)
    return Q, R, perm


def least_squares(A, B):
    """core.py:297-325 (overdetermined branch: pivoted-QR basic solution
    with truncated back substitution; underdetermined: minimum norm)."""
    A = np.asarray(A)
    B = np.asarray(B)
    vec = B.ndim == 1
    B2 = B[:, None] if vec else B
    m, n = A.shape
    if m >= n:
        Q, R, perm = pivoted_qr_r(A)
        Yp = solve_triangular_trunc(R, Q.conj().T @ B2)
        X = np.zeros((n, B2.shape[1]), dtype=Yp.dtype)
        X[perm[:Yp.shape[0]], :] = Yp
    else:
        X = np.linalg.pinv(A) @ B2
    return X[:, 0] if vec else X


def svd_one_pass_general(bundle):
    """factor.py:364-401: dense least squares over vec(B)."""
    Q, Qt = bundle.Q, bundle.Q_tilde
    k, kt = Q.shape[1], Qt.shape[1]
    if k * kt > ONE_PASS_DIM_CAP:
        raise ValueError(f"reduced problem has {k * kt} unknowns, above the cap "
                         f"{ONE_PASS_DIM_CAP}; use the two-pass path")
    if k == 0 or kt == 0:
        dt = bundle.Y.dtype
        return PartialSVD(U=np.zeros((Q.shape[0], 0), dt), sigma=np.zeros(0),
                          V=np.zeros((Qt.shape[0], 0), dt))
    P = Qt.conj().T @ bundle.Omega
    N1 = Q.conj().T @ bundle.Y
    S = Q.conj().T @ bundle.Omega_tilde
    N2 = Qt.conj().T @ bundle.Y_tilde
    dt = np.promote_types(P.dtype, N1.dtype)
    M_top = np.kron(P.T, np.eye(k, dtype=dt))
    M_bot = np.kron(np.eye(kt, dtype=dt), S.conj().T)
    rhs = np.concatenate([N1.reshape(-1, order="F"), N2.conj().T.reshape(-1, order="F")])
    B = least_squares(np.vstack([M_top, M_bot]), rhs).reshape((k, kt), order="F")
    f = small_svd(B)
    return PartialSVD(U=Q @ f.U, sigma=f.sigma, V=Qt @ f.V)


def eig_one_pass(bundle):
    """factor.py:338-361."""
    Q = bundle.Q
    M = Q.conj().T @ bundle.Omega
    N = Q.conj().T @ bundle.Y
    B = least_squares(M.conj().T, N.conj().T).conj().T
    B = 0.5 * (B + B.conj().T)
    diagnostics = {"q_choice": bundle.q_choice}
    sv = small_svd(M).sigma
    tau_min = float(sv.min()) if sv.size else 0.0
    diagnostics["tau_min"] = tau_min
    if sv.size and (tau_min == 0.0 or sv.max() / max(tau_min, 1e-300) > ONE_PASS_COND_WARN):
        diagnostics["ill_conditioned"] = True
    V, lam = small_eig_hermitian(B)
    return PartialEig(U=Q @ V, lam=lam, diagnostics=diagnostics)


# ---------------------------------------------------------------------------
# Interpolative decomposition and row extraction (reference factor.py:198-296)

def pivoted_qr_full(A, max_rank=None):
    """Businger-Golub column-pivoted Householder QR, norms recomputed every
    step, ties to the lowest position (core.py:133-186): (Rp in pivoted
    order k x n with a real nonnegative diagonal, perm)."""
    W = np.array(A, dtype=np.complex128 if np.iscomplexobj(A) else np.float64)
    m, n = W.shape
    steps = min(m, n) if max_rank is None else min(max_rank, m, n)
    perm = np.arange(n)
    for j in range(steps):
        norms = np.linalg.norm(W[j:, j:], axis=0)
        piv = int(np.argmax(norms)) + j
        if piv != j:
            W[:, [j, piv]] = W[:, [piv, j]]
            perm[[j, piv]] = perm[[piv, j]]
        x = W[j:, j]
        xnorm = np.linalg.norm(x)
        if xnorm > 0:
            ph = x[0] / abs(x[0]) if abs(x[0]) > 0 else 1.0
            v = x.copy()
            v[0] += ph * xnorm
            vnorm = np.linalg.norm(v)
            if vnorm > 0:
                v = v / vnorm
                W[j:, j:] -= 2.0 * np.outer(v, v.conj() @ W[j:, j:])
    Rp = np.triu(W[:steps, :])
    d = np.diagonal(Rp)
    ph = np.ones_like(d)
    nz = np.abs(d) > 0
    ph[nz] = d[nz] / np.abs(d[nz])
    Rp = Rp * np.conj(ph)[:, None]
    return Rp, perm


def _column_id(B, k, trunc_tol=TRIANGULAR_TRUNC_TOL):
    """factor.py:198-229 (with the Gu-Eisenstat refinement)."""
    B = np.asarray(B)
    n = B.shape[1]
    Rp, perm0 = pivoted_qr_full(B, max_rank=k)
    perm = list(perm0)
    cap = max(int(3 * k * math.log(max(n, 2))), 8)

    def coefficients(order):
        R = np.linalg.qr(B[:, order], mode="r")
        return solve_triangular_trunc(R[:k, :k], R[:k, k:], trunc_tol=trunc_tol)

    T = solve_triangular_trunc(Rp[:k, :k], Rp[:k, k:], trunc_tol=trunc_tol)
    swaps = 0
    while T.size and np.abs(T).max() > 2.0 * (1.0 + 1e-12):
        i, j = np.unravel_index(int(np.argmax(np.abs(T))), T.shape)
        perm[i], perm[k + j] = perm[k + j], perm[i]
        T = coefficients(perm)
        swaps += 1
        if swaps > cap:
            raise RuntimeError("interpolative decomposition refinement did not settle")
    return np.asarray(perm[:k]), np.asarray(perm[k:]), T


def row_id(M, k):
    """factor.py:232-246: M ~= X M[J, :]."""
    M = np.asarray(M)
    J, free, T = _column_id(M.conj().T, k)
    X = np.zeros((M.shape[0], k), dtype=np.promote_types(T.dtype, M.dtype))
    X[J, :] = np.eye(k)
    X[free, :] = T.conj().T
    return J, X


def householder_qr(A):
    """core.py:67-81 (economy, diagonal of R real nonnegative)."""
    Q, R = np.linalg.qr(np.asarray(A), mode="reduced")
    k = min(np.shape(A))
    d = np.diagonal(R)[:k]
    ph = np.ones_like(d)
    nz = np.abs(d) > 0
    ph[nz] = d[nz] / np.abs(d[nz])
    Q[:, :k] *= ph
    R[:k, :] *= np.conj(ph)[:, None]
    return Q, R


def svd_via_row_extraction(A, QorY):
    """factor.py:267-281."""
    A = np.asarray(A)
    QorY = np.asarray(QorY)
    k = QorY.shape[1]
    J, X = row_id(QorY, k)
    W, Rh = householder_qr(A[J, :].conj().T)
    f = small_svd(X @ Rh.conj().T)
    return PartialSVD(U=f.U, sigma=f.sigma, V=W @ f.V)
