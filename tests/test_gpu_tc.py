"""Round-2 tensor-core kernels against fp64 references: the CTA-pair
persistent fp32 pass (gemm_f32_pair_kernel) over awkward shapes, split-K
remainders and both operand orders, bit-equality with itself run to run,
agreement with the single-CTA kernel (LR_TC_PAIR=0); and the tcgen05 Gram of
an fp32 panel (lr_gram_tc) used by the second CholeskyQR pass."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _pass(A, X, adjoint):
    from paper_0909_4061_b200 import core
    rows = A.shape[1] if adjoint else A.shape[0]
    Y = torch.empty((rows, X.shape[1]), dtype=A.dtype, device=A.device)
    core._pass(A, X, Y, adjoint, float(A.abs().max()))
    return Y


@pytest.mark.parametrize("m,n,ell", [(256, 64, 256), (300, 100, 32), (1000, 333, 17),
                                     (4096, 2048, 256), (257, 4000, 130), (20000, 512, 110),
                                     (70000, 256, 256), (129, 9000, 48)])
@pytest.mark.parametrize("adjoint", [False, True])
def test_pair_pass_vs_fp64(m, n, ell, adjoint):
    g = torch.Generator(device="cuda").manual_seed(m + n + ell)
    A = torch.randn(m, n, device="cuda", generator=g)
    X = torch.randn(m if adjoint else n, ell, device="cuda", generator=g)
    X[:, ::3] *= 1e-3                       # per-column scales differ
    Y = _pass(A, X, adjoint)
    Ad, Xd = A.double(), X.double()
    ref = (Ad.T @ Xd) if adjoint else (Ad @ Xd)
    bound = (Ad.abs().T @ Xd.abs()) if adjoint else (Ad.abs() @ Xd.abs())
    err = ((Y.double() - ref).abs() / bound.clamp_min(1e-300)).max().item()
    assert err <= 2e-6
    Y2 = _pass(A, X, adjoint)
    assert torch.equal(Y, Y2)


@pytest.mark.parametrize("adjoint", [False, True])
def test_pair_matches_single_cta_kernel(adjoint, monkeypatch):
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(9000, 1500, device="cuda", generator=g)
    X = torch.randn(9000 if adjoint else 1500, 200, device="cuda", generator=g)
    Y = _pass(A, X, adjoint)
    monkeypatch.setenv("LR_TC_PAIR", "0")
    Y1 = _pass(A, X, adjoint)
    Ad, Xd = A.double(), X.double()
    ref = (Ad.T @ Xd) if adjoint else (Ad @ Xd)
    bound = (Ad.abs().T @ Xd.abs()) if adjoint else (Ad.abs() @ Xd.abs())
    assert ((Y.double() - ref).abs() / bound).max().item() <= 2e-6
    assert ((Y1.double() - ref).abs() / bound).max().item() <= 2e-6


@pytest.mark.parametrize("m,ell", [(4096, 20), (50000, 128), (70001, 200), (2 ** 20, 256)])
def test_gram_tc(m, ell):
    """lr_gram_tc on a near-orthonormal panel: fp32-level accuracy (the
    second CholeskyQR pass), symmetric, and the overflow flag."""
    from paper_0909_4061_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(ell)
    Y = torch.randn(m, ell, device="cuda", generator=g) / np.sqrt(m)
    G = torch.empty(ell, ell, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    h = _lib.handle()
    _lib.call("lr_gram_tc", h, m, ell, _lib.ptr(Y), ell, _lib.ptr(G), 12, _lib.ptr(st))
    ref = Y.double().T @ Y.double()
    assert int(st.item()) == 0
    assert torch.equal(G, G.T)
    d = torch.diagonal(G) - torch.diagonal(ref)
    assert d.abs().max().item() <= 1e-12 * torch.diagonal(ref).max().item()   # exact fp64 diagonal
    off = (G - ref) - torch.diag(d)
    assert off.abs().max().item() <= 1e-6 * torch.diagonal(ref).max().item()
    Y[7, 3] = 100.0                                  # 100 * 2^12 > 2^15
    _lib.call("lr_gram_tc", h, m, ell, _lib.ptr(Y), ell, _lib.ptr(G), 12, _lib.ptr(st))
    assert int(st.item()) & 1


def test_fp32_orth_second_pass_on_tc(monkeypatch):
    """The fp32 CholeskyQR2 with its second Gram on the tensor cores gives an
    orthonormal Q (to fp32 level) spanning the same space as with the exact
    Gram (LR_GRAM_TC=0)."""
    from paper_0909_4061_b200 import core
    g = torch.Generator(device="cuda").manual_seed(9)
    m, ell = 200000, 256
    Y = torch.randn(m, ell, device="cuda", generator=g) @ torch.diag(
        torch.logspace(0, -5, ell, device="cuda"))
    Q = core.orth_dev(Y)
    monkeypatch.setenv("LR_GRAM_TC", "0")
    Q0 = core.orth_dev(Y)
    I = torch.eye(ell, dtype=torch.float64, device="cuda")
    assert (Q.double().T @ Q.double() - I).abs().max().item() <= 5e-6
    assert (Q0.double().T @ Q0.double() - I).abs().max().item() <= 5e-6
    assert (Q.double() - Q0.double()).abs().max().item() <= 1e-4


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("m,ell", [(4096, 256), (70001, 200), (300000, 130), (2 ** 20, 256),
                                   (20000, 64), (8192, 300)])
def test_exact_gram_symmetric_tiles(m, ell, dtype):
    """lr_gram (the exact DMMA Gram of the first CholeskyQR pass): diagonal
    CTA tiles skip the warps strictly below the diagonal and the lower
    triangle is mirrored -- the whole matrix equals an fp64 product of the
    same panel to fp64 roundoff and is exactly symmetric."""
    from paper_0909_4061_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(m + ell)
    Y = torch.randn(m, ell, device="cuda", generator=g, dtype=dtype)
    Y[:, 1::4] *= 1e-3
    G = torch.empty(ell, ell, dtype=torch.float64, device="cuda")
    code = _lib.F32 if dtype == torch.float32 else _lib.F64
    _lib.call("lr_gram", _lib.handle(), code, m, ell, _lib.ptr(Y), ell, _lib.ptr(G))
    Yd = Y.double()
    ref = Yd.T @ Yd
    bound = Yd.abs().T @ Yd.abs()
    assert torch.equal(G, G.T)
    assert ((G - ref).abs() / bound).max().item() <= 1e-13
