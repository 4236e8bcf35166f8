"""Structured sketches on the GPU: the radix-16 Stockham FFT SRFT, the
reference's operation counter and acceptance #15 (tests/test_acceptance.py:
386-421), sketch_apply / dense_sketch_matrix (sketch.py:340-358), and the CLI
Stage-A dispatch with the SRFT doubling ladder (cli.py:128-165)."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def lr():
    import paper_0909_4061_b200 as m
    return m


@pytest.mark.parametrize("n", [256, 512, 2048, 4096, 8192, 16384])
@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_srft16_vs_oracle(n, dtype, monkeypatch):
    """Every radix mix of the Stockham kernel (16^p x {1, 2, 4, 8}) against
    the oracle's SRFT, and against the radix-2 kernel (LR_SRFT=radix2)."""
    from oracle import lowrank_oracle as O
    rng = np.random.default_rng(n)
    A = (rng.standard_normal((37, n)) + 1j * rng.standard_normal((37, n))).astype(dtype)
    ell = 24
    op = lr().srft_operator(n, ell, 5)
    Y = lr().srft_apply(A, op)
    Yo = O.srft_apply(A.astype(np.complex128), O.srft_operator(n, ell, 5))
    tol = 2e-5 if dtype == np.complex64 else 1e-12
    assert np.abs(Y - Yo).max() <= tol * np.abs(Yo).max()
    if dtype == np.complex128 and n == 16384:
        return     # beyond the shared-memory FFTs: the dense path either way
    monkeypatch.setenv("LR_SRFT", "radix2")
    Y2 = lr().srft_apply(A, op)
    assert np.abs(Y - Y2).max() <= tol * np.abs(Yo).max()


@pytest.mark.parametrize("n", [2, 16, 256, 4096])
def test_dft_matches_numpy(n):
    rng = np.random.default_rng(n + 1)
    x = rng.standard_normal((5, n)) + 1j * rng.standard_normal((5, n))
    y = lr().dft(x)
    assert np.abs(y - np.fft.fft(x, axis=-1) / np.sqrt(n)).max() <= 1e-12 * np.sqrt(n)


def test_acceptance_15_correctness_and_complexity():
    """Reference acceptance #15: the fast path equals the dense product on
    mixed sizes, and the operation counter stays below 8 m n log2 n with an
    n-exponent in [0.9, 1.2]."""
    m_ = lr()
    worst = 0.0
    rng = np.random.default_rng(1515)
    for n in (12, 100, 256, 1000):
        A = rng.standard_normal((8, n))
        om = m_.srft_operator(n, min(6, n), seed=n)
        fast = m_.srft_apply(A, om)
        dense = A @ om.to_dense()
        worst = max(worst, np.abs(fast - dense).max() / max(1.0, np.abs(dense).max()))
    assert worst <= 1e-11
    m, ell = 4, 8
    ns = [256, 512, 1024, 2048, 4096]
    counts = []
    for n in ns:
        A = m_.gaussian_matrix(n, m, seed=n).T
        m_.reset_op_count()
        m_.srft_apply(A, m_.srft_operator(n, ell, seed=n + 1))
        counts.append(m_.op_count())
    slope = np.polyfit(np.log(ns), np.log(counts), 1)[0]
    assert 0.9 <= slope <= 1.2
    assert all(c <= 8 * m * n * math.log2(n) for c, n in zip(counts, ns))


def test_sketch_apply_and_dense_matrix():
    """sketch.py:340-358: sketch_apply(A, spec) == A @ dense_sketch_matrix."""
    m_ = lr()
    rng = np.random.default_rng(3)
    A = rng.standard_normal((20, 64))
    for kind in ("gaussian", "srft", "gsrft"):
        spec = m_.SketchSpec(kind=kind, ell=7, seed=4)
        Y = m_.sketch_apply(A, spec)
        Om = m_.dense_sketch_matrix(64, spec)
        assert Om.shape == (64, 7)
        assert np.abs(Y - A @ Om).max() <= 1e-12 * np.abs(A @ Om).max()
    assert np.array_equal(m_.dense_sketch_matrix(64, m_.SketchSpec("gaussian", 7, seed=4)),
                          m_.gaussian_matrix(64, 7, 4))


def test_stage_a_srft_ladder_vs_oracle():
    """cli.py:139-150: ell = 32, 64, 128, ... with the estimate at seed + 7
    until it meets tol -- same final ell, saturation flag and estimate as the
    oracle's restatement of the ladder."""
    from oracle import lowrank_oracle as O
    m_ = lr()
    rng = np.random.default_rng(7)
    U = np.linalg.qr(rng.standard_normal((300, 120)))[0]
    V = np.linalg.qr(rng.standard_normal((256, 120)))[0]
    A = (U * np.exp(-np.arange(120) / 12.0)) @ V.T
    for tol in (1e-1, 1e-3, 1e-12):
        basis, _ = m_.stage_a(A, sketch="srft", tol=tol, seed=2)
        ell = 32
        while True:
            ell = min(ell, 256)
            ob = O.fast_range_finder(A, ell, 2, kind="srft")
            est = O.posterior_error_estimate(O.Dense(A), ob.Q, seed=2 + 7)
            if est <= tol or ell >= 256:
                break
            ell *= 2
        assert basis.samples_used == ell
        assert basis.est_error == pytest.approx(est, rel=1e-6)
        assert basis.saturated == (ell >= 256 and est > tol)
    with pytest.raises(ValueError):
        m_.stage_a(A, sketch="srft", rank=10, power=1)
    with pytest.raises(ValueError):
        m_.stage_a(A, adaptive=True)
    b, _ = m_.stage_a(A, rank=20, oversample=5, power=1, seed=3)
    assert b.passes == 4 and b.Q.shape[1] == 25


def test_svd_single_pass_composition():
    from oracle import lowrank_oracle as O
    m_ = lr()
    rng = np.random.default_rng(11)
    A = (rng.standard_normal((90, 15)) * np.exp(-np.arange(15))) @ rng.standard_normal((15, 70))
    f, est = m_.svd_single_pass(A, 10, 5, seed=4)
    b = O.sample_bundle_two_sided(A, 15, seed=4)
    fo = O.svd_one_pass_general(b)
    esto = O.posterior_error_estimate(O.Dense(A), b.Q, seed=4 + 13)
    assert np.abs(f.sigma - fo.sigma).max() <= 1e-10 * fo.sigma[0]
    assert est == pytest.approx(esto, rel=1e-6)
