"""Hermitian Stage-B routes on the GPU (reference factor.py:168-191,300-335,
core.py:233-294) against the reference's golden vectors and
the CPU oracle."""

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


def test_direct_eig_golden(golden):
    g = golden("stageb")
    m = lr()
    for key in ("eig", "eigc"):
        f = m.direct_eig_hermitian(g[f"{key}_A"], g[f"{key}_Q"])
        scale = np.abs(g[f"{key}_lam"]).max()
        assert np.abs(f.lam - g[f"{key}_lam"]).max() <= 1e-12 * scale
        assert np.abs(f.compose() - g[f"{key}_comp"]).max() <= 1e-12 * scale
        assert np.linalg.norm(f.U.conj().T @ f.U - np.eye(f.U.shape[1])) <= 1e-12
    f = m.direct_eig_hermitian(np.diag([3.0, -2.0, 1.0]), np.eye(3))
    assert np.allclose(f.lam, g["eig_diag_lam"], rtol=0, atol=1e-14)


def test_small_eig_hermitian_golden_and_order(golden):
    g = golden("stageb")
    m = lr()
    V, lam = m.small_eig_hermitian(g["seig_B"])
    assert np.abs(lam - g["seig_lam"]).max() <= 1e-13 * np.abs(lam).max()
    H = 0.5 * (g["seig_B"] + g["seig_B"].T)
    assert np.abs((V * lam) @ V.T - H).max() <= 1e-13 * np.abs(H).max()
    # ties: equal magnitudes in descending value (core.py:245)
    V, lam = m.small_eig_hermitian(np.diag([2.0, -2.0, 1.0, 0.0]))
    assert np.allclose(lam, [2.0, -2.0, 1.0, 0.0], rtol=0, atol=1e-14)
    V, lam = m.small_eig_hermitian(np.zeros((4, 4)))
    assert np.abs(lam).max() <= 1e-15


def test_direct_eig_rejects_non_hermitian():
    m = lr()
    A = np.random.default_rng(13).standard_normal((10, 10))
    with pytest.raises(ValueError):
        m.direct_eig_hermitian(A, np.eye(10)[:, :3])


@pytest.mark.parametrize("dtype", [np.float64, np.complex128, np.float32])
def test_direct_eig_vs_oracle(dtype):
    """n = 3000 Hermitian with a decaying spectrum of both signs, basis from
    the device range finder; eigenvalues, reconstruction and counters (the
    probe's two applications + the B pass) against the oracle."""
    from oracle import lowrank_oracle as O
    m = lr()
    g = np.random.default_rng(5)
    n, ell = 3000, 40
    X = g.standard_normal((n, n)) + (1j * g.standard_normal((n, n)) if dtype == np.complex128 else 0)
    U = np.linalg.qr(X)[0][:, :200]
    lam0 = np.exp(-np.arange(200) / 15.0) * np.where(np.arange(200) % 3 == 1, -1.0, 1.0)
    A = ((U * lam0) @ U.conj().T).astype(dtype)
    A = 0.5 * (A + A.conj().T)
    Q = m.randomized_range_finder(A, ell, seed=3).Q
    op = m.DenseOperator(A)
    f = m.direct_eig_hermitian(op, Q)
    fo = O.direct_eig_hermitian(A.astype(np.complex128 if dtype == np.complex128 else np.float64),
                                Q.astype(np.complex128 if dtype == np.complex128 else np.float64))
    tol = 1e-11 if dtype != np.float32 else 2e-5
    assert np.abs(f.lam - fo.lam).max() <= tol * np.abs(fo.lam).max()
    assert np.abs(f.compose() - fo.compose()).max() <= tol * np.abs(fo.lam).max()
    assert op.counters.passes == 3 and op.counters.matvecs == 2 + ell


def test_nystrom_golden(golden):
    g = golden("stageb")
    m = lr()
    for tag in ("nys_rank", "nys_exp", "nys_pow"):
        f, fac = m.eig_nystrom(g[f"{tag}_H"], g[f"{tag}_Q"])
        scale = np.abs(g[f"{tag}_lam"]).max()
        assert np.abs(f.lam - g[f"{tag}_lam"]).max() <= 1e-10 * scale, tag
        assert np.abs(f.compose() - g[f"{tag}_comp"]).max() <= 1e-10 * scale, tag
        assert np.abs(fac.F @ fac.F.conj().T - g[f"{tag}_FF"]).max() <= 1e-10 * scale, tag
        assert np.all(f.lam >= 0) and not f.diagnostics
    f, _ = m.eig_nystrom(np.diag([1.0, 0.5, -0.8]), np.eye(3))
    assert f.diagnostics.get("not_psd_fallback")
    assert f.diagnostics["min_projected_eigenvalue"] == pytest.approx(-0.8, abs=1e-12)
    assert np.allclose(f.lam, g["nys_fb_lam"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("dtype", [np.float64, np.complex128])
def test_nystrom_vs_oracle(dtype):
    from oracle import lowrank_oracle as O
    m = lr()
    g = np.random.default_rng(7)
    n, ell = 2500, 30
    X = g.standard_normal((n, 300)) + (1j * g.standard_normal((n, 300)) if dtype == np.complex128 else 0)
    U = np.linalg.qr(X)[0]
    H = ((U * np.exp(-np.arange(300) / 8.0)) @ U.conj().T).astype(dtype)
    H = 0.5 * (H + H.conj().T)
    Q = m.randomized_range_finder(H, ell, seed=11).Q
    f, fac = m.eig_nystrom(H, Q)
    fo, F = O.eig_nystrom(H, Q)
    assert np.abs(f.lam - fo.lam).max() <= 1e-10 * fo.lam.max()
    assert np.abs(f.compose() - fo.compose()).max() <= 1e-10 * fo.lam.max()
    # never exceeds the basis residual (reference test_factor.py:238-244)
    eps = np.linalg.norm(H - Q @ (Q.conj().T @ H), 2)
    assert np.linalg.norm(H - f.compose(), 2) <= eps * (1 + 1e-9) + 1e-12
