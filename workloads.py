"""Seeded synthetic inputs for BASELINE.json's five configurations.

Neither product code nor oracle: these builders produce the matrices that
tests/ and bench.py feed to both the CUDA path and the CPU oracle.  The
paper's data-dependent experiments (image graph Laplacian, FERET faces) are
not available offline; seeded synthetic matrices with the configs' shapes,
spectra and value distributions stand in for them.

Recipes (all randomness from the reference's Philox keying, reference
sketch.py:32-42, unless a builder says otherwise):

  cfg1  fp64 2048^2, A = U diag(s) V^T, s_j = exp(-(j-1)/20)   -- reference
        oracle.py:114-126 synthetic_matrix (U then V from stream "synt").
  cfg2  fp64 16384x8192, same builder, s_j = j^-1/2.
  cfg3  complex64 8192^2, A = N + P: N i.i.d. complex Gaussian
        (re, im ~ N(0, 1/2), stream "nois"); P = G1 G2^H with G1, G2 complex
        Gaussian 8192x50 (stream "plnt"), scaled so ||P||_F = 100 ||N||_F.
  cfg4  fp32 2^20 x 4096, A = U diag(s) V^T built in fp64, stored fp32:
        U = vstack_b haar(65536, 4096, rng(s, "Ublk", b)) / sqrt(#blocks),
        V = haar(4096, 4096, rng(s, "Vhar")), s_j = 0.9^(j-1) (j <= 200)
        else 1e-6.  The full-size device build draws the same Philox streams
        on the GPU (numpy-matching generator) and QR-factors them there.
  cfg5  fp64 CSR 2^21 x 2^21 with 16 uniform random columns per row
        (duplicates summed), values N(0,1) (stream "sprs"); plus implicit
        L R^T with L, R = 10 * Gaussian n x 32 (stream "lowr").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

STREAM_SYNTH = 0x73796E74   # "synt", reference oracle.py:120
STREAM_NOISE = 0x6E6F6973   # "nois"
STREAM_PLANT = 0x706C6E74   # "plnt"
STREAM_UBLK = 0x55626C6B    # "Ublk"
STREAM_VHAR = 0x56686172    # "Vhar"
STREAM_SPRS = 0x73707273    # "sprs"
STREAM_LOWR = 0x6C6F7772    # "lowr"

# nonzeros of the cfg5 recipe at seed 5 (duplicates summed), SURVEY.md §8d
CFG5_NNZ = 33554314


def rng_for(seed, stream=0, index=0):
    """Reference sketch.py:32-42 Philox keying (restated; see oracle)."""
    key = (int(seed) % (1 << 64)) | ((int(stream) % (1 << 32)) << 64) | (
        (int(index) % (1 << 32)) << 96)
    return np.random.Generator(np.random.Philox(key=key))


@dataclass(frozen=True)
class Config:
    idx: int
    name: str
    m: int
    n: int
    dtype: str
    k: int
    p: int
    q: int
    sketch: str = "gauss"

    @property
    def ell(self):
        return self.k + self.p

    @property
    def seed(self):
        return self.idx

    def passes(self):
        """Passes over A for Stage A + direct SVD: 2q+2 (reference
        rangefinder.py:217,242 convention; Alg 4.1/4.5 + Alg 5.1 = 2)."""
        return 2 * self.q + 2

    def a_bytes(self, nnz=None):
        if self.idx == 5:
            # CSR bytes model: f64 values + int32 columns + int64 row pointers
            nnz = CFG5_NNZ if nnz is None else nnz
            return nnz * 12 + (self.m + 1) * 8
        elem = {"f64": 8, "f32": 4, "c64": 8, "c128": 16}[self.dtype]
        return self.m * self.n * elem


CONFIGS = {
    1: Config(1, "dense-f64-2048-gauss-q0", 2048, 2048, "f64", 20, 10, 0),
    2: Config(2, "dense-f64-16384x8192-subspace-q2", 16384, 8192, "f64", 100, 10, 2),
    3: Config(3, "dense-c64-8192-srft", 8192, 8192, "c64", 50, 70, 0, "srft"),
    4: Config(4, "dense-f32-1Mx4096-rowsharded-q1", 1 << 20, 4096, "f32", 200, 56, 1),
    5: Config(5, "csr-f64-2M-plus-lowrank-q3", 1 << 21, 1 << 21, "f64", 32, 16, 3),
}


# ---------------------------------------------------------------------------
# spectra

def spectrum(cfg_idx, r):
    j = np.arange(1, r + 1, dtype=np.float64)
    if cfg_idx == 1:
        s = np.exp(-(j - 1) / 20.0)
    elif cfg_idx == 2:
        s = j ** -0.5
    elif cfg_idx == 4:
        s = np.where(j <= 200, 0.9 ** (j - 1), 1e-6)
    else:
        raise ValueError(cfg_idx)
    return s


# ---------------------------------------------------------------------------
# host (numpy) builders -- reference recipes, usable at reduced sizes

def haar_basis(rows, cols, rng):
    """Reference oracle.py:107-111: Q of a Gaussian, columns signed by diag R."""
    g = rng.standard_normal((rows, cols))
    q, r = np.linalg.qr(g, mode="reduced")
    d = np.diagonal(r)
    return q * np.where(np.abs(d) > 0, np.sign(d), 1.0)


def synthetic_explicit(m, n, s, seed):
    """Reference oracle.py:114-126 with kind="explicit" (s sorted descending,
    oracle.py:101): U then V from one stream."""
    r = min(m, n)
    sv = np.zeros(r)
    sv[:min(r, len(s))] = np.asarray(s, dtype=np.float64)[:r]
    sv = np.sort(sv)[::-1]
    rng = rng_for(seed, STREAM_SYNTH)
    U = haar_basis(m, r, rng)
    V = haar_basis(n, r, rng)
    return (U * sv) @ V.T, sv


def build_cfg1(seed=1, m=2048, n=2048):
    return synthetic_explicit(m, n, spectrum(1, min(m, n)), seed)


def build_cfg3(seed=3, m=8192, n=8192, rank=50, ratio=100.0):
    g = rng_for(seed, STREAM_NOISE)
    N = (g.standard_normal((m, n)) + 1j * g.standard_normal((m, n))) * np.sqrt(0.5)
    h = rng_for(seed, STREAM_PLANT)
    G1 = (h.standard_normal((m, rank)) + 1j * h.standard_normal((m, rank))) * np.sqrt(0.5)
    G2 = (h.standard_normal((n, rank)) + 1j * h.standard_normal((n, rank))) * np.sqrt(0.5)
    P = G1 @ G2.conj().T
    P *= ratio * np.linalg.norm(N) / np.linalg.norm(P)
    return (N + P).astype(np.complex64)


def build_cfg4_host(seed=4, m=65536, n=4096, block=65536):
    """Reduced-row cfg4 on the host (m a multiple of `block`)."""
    nb = m // block
    s = spectrum(4, n)
    V = haar_basis(n, n, rng_for(seed, STREAM_VHAR))
    W = (V * s).T            # diag(s) V^T
    A = np.empty((m, n), dtype=np.float32)
    for b in range(nb):
        Ub = haar_basis(block, n, rng_for(seed, STREAM_UBLK, b)) / np.sqrt(nb)
        A[b * block:(b + 1) * block] = (Ub @ W).astype(np.float32)
    return A, s


def build_cfg5(seed=5, n=1 << 21, per_row=16, rank=32, scale=10.0):
    """CSR S (row pointers int64, columns int32, values f64) plus L, R."""
    import scipy.sparse as sp
    g = rng_for(seed, STREAM_SPRS)
    cols = g.integers(0, n, size=(n, per_row)).astype(np.int64)
    vals = g.standard_normal((n, per_row))
    rows = np.repeat(np.arange(n, dtype=np.int64), per_row)
    S = sp.csr_matrix((vals.ravel(), (rows, cols.ravel())), shape=(n, n))
    S.sum_duplicates()
    S.sort_indices()
    h = rng_for(seed, STREAM_LOWR)
    L = scale * h.standard_normal((n, rank))
    R = scale * h.standard_normal((n, rank))
    return S, L, R


# ---------------------------------------------------------------------------
# device (torch) builders for full-size timing runs

def _haar_torch(g, device):
    import torch
    q, r = torch.linalg.qr(g)
    d = torch.diagonal(r)
    sgn = torch.where(d.abs() > 0, torch.sign(d), torch.ones_like(d))
    return q * sgn


def build_synthetic_device(m, n, s, seed, device="cuda", host_rng=True):
    """cfg1/cfg2 recipe on the GPU: the reference's Gaussian draws (host
    Philox, identical stream order) are uploaded and QR-factored on the
    device in fp64; A = (U * s) @ V^T in fp64.  Differs from the host build
    only by QR rounding (~1e-15 relative)."""
    import torch
    r = min(m, n)
    sv = torch.zeros(r, dtype=torch.float64)
    sv[:min(r, len(s))] = torch.as_tensor(np.sort(np.asarray(s, np.float64)[:r])[::-1].copy())
    if host_rng:
        rng = rng_for(seed, STREAM_SYNTH)
        gu = torch.from_numpy(rng.standard_normal((m, r))).to(device)
        U = _haar_torch(gu, device)
        del gu
        gv = torch.from_numpy(rng.standard_normal((n, r))).to(device)
    else:
        gen = torch.Generator(device=device).manual_seed(seed)
        gu = torch.randn((m, r), dtype=torch.float64, device=device, generator=gen)
        U = _haar_torch(gu, device)
        del gu
        gv = torch.randn((n, r), dtype=torch.float64, device=device, generator=gen)
    V = _haar_torch(gv, device)
    del gv
    A = (U * sv.to(device)) @ V.T
    return A, sv.numpy()


def build_cfg4_device(seed=4, m=1 << 20, n=4096, block=65536, device="cuda", rows=None):
    """Full-size cfg4 on the GPU with the exact recipe of build_cfg4_host:
    the Gaussian blocks are the reference's Philox streams rng_for(seed,
    "Ublk", b) / rng_for(seed, "Vhar") drawn on the device by the library's
    numpy-matching generator (lr_gaussian, checked against numpy in
    tests/test_gpu_kernels.py), QR-factored in fp64 on the device (cuSOLVER
    Householder, like numpy's LAPACK QR up to roundoff) and signed by diag R;
    A = U diag(s) V^T in fp64, stored fp32.  Differs from the host build only
    by fp64 QR rounding (~1e-15 relative), i.e. at most one fp32 ulp on rare
    entries (tests/test_gpu_parity.py checks a block against the host).
    rows=(r0, r1): build only those rows (a rank's shard), same values."""
    import torch
    from paper_0909_4061_b200.sketch import gaussian_dev
    nb = m // block
    dev = torch.device(device)
    s = torch.as_tensor(spectrum(4, n), dtype=torch.float64, device=dev)
    V = _haar_torch(gaussian_dev(n, n, seed, stream=STREAM_VHAR, dtype=torch.float64,
                                 device=dev.index), device)
    W = (V * s).T.contiguous()
    del V
    r0, r1 = (0, m) if rows is None else rows
    A = torch.empty((r1 - r0, n), dtype=torch.float32, device=dev)
    for b in range(r0 // block, -(-r1 // block)):
        g = gaussian_dev(block, n, seed, stream=STREAM_UBLK, index=b, dtype=torch.float64,
                         device=dev.index)
        Ub = _haar_torch(g, device) / np.sqrt(nb)
        del g
        lo, hi = max(r0, b * block), min(r1, (b + 1) * block)
        A[lo - r0:hi - r0] = (Ub[lo - b * block:hi - b * block] @ W).to(torch.float32)
        del Ub
    torch.cuda.synchronize(dev)
    return A, s.cpu().numpy()


def cfg4_block_host(b, seed=4, m=1 << 20, n=4096, block=65536):
    """Block b (rows [b*block, (b+1)*block)) of the full-size cfg4 recipe on
    the host (reference haar_basis via numpy QR) -- the recipe check for
    build_cfg4_device."""
    nb = m // block
    s = spectrum(4, n)
    V = haar_basis(n, n, rng_for(seed, STREAM_VHAR))
    Ub = haar_basis(block, n, rng_for(seed, STREAM_UBLK, b)) / np.sqrt(nb)
    return (Ub @ (V * s).T).astype(np.float32)
