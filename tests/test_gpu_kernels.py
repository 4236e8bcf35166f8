"""Kernel-level parity on the GPU: each C-ABI entry point against numpy /
the CPU oracle on seeded inputs (bit-exact where integer, stated tolerance
where floating point)."""

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


def rand(shape, dtype, seed):
    g = np.random.default_rng(seed)
    a = g.standard_normal(shape)
    if np.dtype(dtype).kind == "c":
        a = a + 1j * g.standard_normal(shape)
    return a.astype(dtype)


GEMM_SHAPES = [(300, 257, 30), (1, 5, 1), (129, 64, 110), (64, 1000, 10), (513, 77, 128),
               (200, 300, 130), (2048, 2048, 30), (37, 1, 3)]


@pytest.mark.parametrize("m,n,ell", GEMM_SHAPES)
@pytest.mark.parametrize("dtype", [np.float64, np.complex128])
def test_gemm_f64_family(m, n, ell, dtype):
    from paper_0909_4061_b200.core import DenseOperator
    A = rand((m, n), dtype, m + n)
    X = rand((n, ell), dtype, ell)
    W = rand((m, ell), dtype, ell + 1)
    op = DenseOperator(A)
    Y = op.apply(X)
    ref = A @ X
    scale = np.abs(A).max() * np.abs(X).max() * n
    assert np.abs(Y - ref).max() <= 1e-14 * scale
    Z = op.apply_adjoint(W)
    ref = A.conj().T @ W
    assert np.abs(Z - ref).max() <= 1e-14 * np.abs(A).max() * np.abs(W).max() * m
    assert op.counters.passes == 2 and op.counters.matvecs == ell


@pytest.mark.parametrize("m,n,ell", [(300, 257, 30), (129, 64, 110), (1000, 512, 64)])
@pytest.mark.parametrize("dtype", [np.float32, np.complex64])
def test_gemm_f32_family(m, n, ell, dtype):
    from paper_0909_4061_b200.core import DenseOperator
    A = rand((m, n), dtype, m + n)
    X = rand((n, ell), dtype, ell)
    op = DenseOperator(A)
    Y = op.apply(X)
    wide = np.complex128 if A.dtype.kind == "c" else np.float64
    ref = A.astype(wide) @ X
    # fp32-level: relative to |A||X| (the tensor-core accumulation truncates)
    bound = np.abs(A).astype(np.float64) @ np.abs(X).astype(np.float64)
    assert (np.abs(Y - ref) / bound).max() <= 4e-6
    W = rand((m, ell), dtype, 3)
    Z = op.apply_adjoint(W)
    ref = A.conj().T.astype(wide) @ W
    bound = np.abs(A).T.astype(np.float64) @ np.abs(W).astype(np.float64)
    assert (np.abs(Z - ref) / bound).max() <= 4e-6


@pytest.mark.parametrize("ell", [1, 10, 20, 30, 48, 110, 130, 256])
@pytest.mark.parametrize("dtype", [np.float32, np.complex64])
def test_tcgen05_pass_shapes(ell, dtype):
    """The fp32 / complex64 passes over A run on tcgen05 (scaled fp16 split);
    every N tile width must agree with fp64 to ~fp32 accuracy."""
    from paper_0909_4061_b200.core import DenseOperator
    m, n = 1536, 1024
    if dtype == np.complex64 and ell > 128:
        pytest.skip("complex real view needs 2 ell <= 256")
    A = rand((m, n), dtype, 11)
    X = rand((n, ell), dtype, 12)
    W = rand((m, ell), dtype, 13)
    op = DenseOperator(A)
    wide = np.complex128 if A.dtype.kind == "c" else np.float64
    Y = op.apply(X)
    ref = A.astype(wide) @ X.astype(wide)
    assert np.abs(Y - ref).max() <= 1e-5 * np.abs(ref).max()
    Z = op.apply_adjoint(W)
    ref = A.astype(wide).conj().T @ W.astype(wide)
    assert np.abs(Z - ref).max() <= 1e-5 * np.abs(ref).max()


@pytest.mark.parametrize("m,n,ell", [(8192, 4096, 20), (1536, 16384, 20), (8192, 16384, 256)])
def test_tcgen05_deep_k_narrow_n(m, n, ell):
    """Long K with a narrow N (tools/tc_probe2.py shapes): the configuration
    where two co-resident CTAs once produced wrong rows."""
    from paper_0909_4061_b200 import core
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(m, n, device="cuda", generator=g)
    X = torch.randn(n, ell, device="cuda", generator=g)
    op = core.DenseOperator(A)
    Y = torch.empty(m, ell, device="cuda")
    core._pass(A, X, Y, False, op.amax)
    ref = A.double() @ X.double()
    assert (Y.double() - ref).abs().max().item() <= 2e-5 * ref.abs().max().item()


def test_gemm_vector_and_strided_inputs():
    from paper_0909_4061_b200.core import DenseOperator
    A = rand((50, 40), np.float64, 1)
    op = DenseOperator(A)
    x = rand(40, np.float64, 2)
    assert op.apply(x).shape == (50,)
    assert np.allclose(op.apply(x), A @ x, rtol=0, atol=1e-13)
    Xt = torch.from_numpy(rand((40, 9), np.float64, 3)).cuda()[:, 2:7]   # strided view
    Y = op.apply(Xt)
    assert torch.is_tensor(Y)
    assert np.allclose(Y.cpu().numpy(), A @ Xt.cpu().numpy(), atol=1e-13)


def test_nonfinite_rejected():
    from paper_0909_4061_b200.core import DenseOperator
    A = np.ones((4, 3))
    A[2, 1] = np.nan
    with pytest.raises(ValueError):
        DenseOperator(A)
    with pytest.raises(ValueError):
        DenseOperator(np.ones((3,)))
    with pytest.raises(ValueError):
        DenseOperator(np.ones((0, 3)))


@pytest.mark.parametrize("m,ell,dtype", [(500, 30, np.float64), (2000, 110, np.float64),
                                         (300, 7, np.complex128), (5000, 256, np.float64),
                                         (1000, 48, np.float32), (400, 20, np.complex64)])
def test_orth_matches_cgs2(m, ell, dtype):
    from oracle import lowrank_oracle as O
    Y = rand((m, ell), dtype, m * ell)
    Q = lr().orthonormalize_double_gs(Y)
    Qo = O.orthonormalize_double_gs(Y.astype(np.complex128 if Y.dtype.kind == "c" else np.float64))
    assert Q.shape == Qo.shape
    tol = 1e-12 if Y.dtype in (np.float64, np.complex128) else 2e-5
    assert np.abs(Q - Qo).max() <= tol
    k = Q.shape[1]
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(k)) <= (1e-12 if tol < 1e-6 else 1e-5) * k


def _chol_drop_ref(G, tol, shift_coef):
    """numpy restatement of the lr_chol_drop contract (column deletion)."""
    n = G.shape[0]
    tr = float(np.real(np.trace(G)))
    thr2 = tol * tol * tr
    W = G.astype(np.complex128 if np.iscomplexobj(G) else np.float64).copy()
    W[np.diag_indices(n)] += shift_coef * tr
    R = np.zeros_like(W)
    kept = []
    for j in range(n):
        d = float(np.real(W[j, j] - sum(abs(R[i, j]) ** 2 for i in kept)))
        if np.isfinite(d) and d > thr2 and d > 0:
            R[j, j] = np.sqrt(d)
            for k in range(j + 1, n):
                R[j, k] = (W[j, k] - sum(np.conj(R[i, j]) * R[i, k] for i in kept)) / R[j, j]
            kept.append(j)
    dropped = [k for k in range(n) if k not in kept]
    R[:, dropped] = 0      # the factor is reported on kept rows/cols only
    return R, kept


@pytest.mark.parametrize("ell,cplx,rank", [(30, False, 30), (100, False, 87), (128, False, 128),
                                           (200, False, 170), (256, False, 256),
                                           (64, True, 50), (120, True, 120), (180, True, 160)])
def test_chol_drop_sizes(ell, cplx, rank):
    """Cholesky with deletion on every kernel path (shared-memory <= 79,
    register-tiled 80..128, 2x2 blocked 129..256): rank decision and
    factor vs a numpy restatement; Q = Y P orthonormal on the kept span."""
    from paper_0909_4061_b200 import _lib
    g = np.random.default_rng(ell)
    m = 3 * ell
    B = g.standard_normal((m, rank)) + (1j * g.standard_normal((m, rank)) if cplx else 0)
    C = g.standard_normal((rank, ell)) + (1j * g.standard_normal((rank, ell)) if cplx else 0)
    Y = B @ C   # exact rank: the first `rank` columns are kept, the rest dropped
    Yd = torch.from_numpy(Y).cuda()
    G = (Yd.conj().T @ Yd).contiguous()
    P, R = torch.empty_like(G), torch.empty_like(G)
    info = torch.zeros(4, dtype=torch.int32, device="cuda")
    code = _lib.C128 if cplx else _lib.F64
    # drop_tol 1e-6: the dependent columns' Gram pivots (~u tr G) are resolvable
    _lib.call("lr_chol_drop", _lib.handle(), code, ell, _lib.ptr(G), 1e-6, 4 * ell * 1.1e-16,
              0.0, _lib.ptr(P), _lib.ptr(R), _lib.ptr(info))
    torch.cuda.synchronize()
    Rref, kept = _chol_drop_ref(G.cpu().numpy(), 1e-6, 0.0)
    r = int(info[0].item())
    assert r == len(kept) == rank
    Rg = R.cpu().numpy()
    scale = np.abs(Rref).max()
    assert np.abs(Rg - Rref).max() <= 1e-9 * scale
    Q = (Yd @ P[:, :r]).cpu().numpy()
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(r)) <= 1e-6 * r
    if r < ell:
        assert np.abs(P[:, r:].cpu().numpy()).max() == 0.0


@pytest.mark.parametrize("ell,cplx", [(17, False), (47, False), (110, False), (199, False),
                                      (230, False), (33, True), (120, True), (140, True),
                                      (150, True)])
@pytest.mark.parametrize("shift", [0.0, 1e-14])   # shift < drop_tol^2: drops stay
def test_chol_drop_interleaved(ell, cplx, shift):
    """Dropped columns scattered through the panel (duplicates of earlier
    columns at panel boundaries and inside panels) and a diagonal shift:
    rank decision, R on the kept rows/cols, and P = R~^{-1} compacted."""
    from paper_0909_4061_b200 import _lib
    g = np.random.default_rng(1000 + ell)
    m = 2 * ell + 5
    Y = g.standard_normal((m, ell)) + (1j * g.standard_normal((m, ell)) if cplx else 0)
    dup = sorted(set(int(x) for x in g.choice(np.arange(1, ell), size=max(1, ell // 9),
                                               replace=False)) | {min(16, ell - 1)})
    for j in dup:       # column j = combination of two earlier columns
        a, b = g.integers(0, j, size=2)
        Y[:, j] = 0.5 * Y[:, a] - 2.0 * Y[:, b]
    Yd = torch.from_numpy(Y).cuda()
    G = (Yd.conj().T @ Yd).contiguous()
    P, R = torch.empty_like(G), torch.empty_like(G)
    info = torch.zeros(4, dtype=torch.int32, device="cuda")
    code = _lib.C128 if cplx else _lib.F64
    _lib.call("lr_chol_drop", _lib.handle(), code, ell, _lib.ptr(G), 1e-6, 4 * ell * 1.1e-16,
              shift, _lib.ptr(P), _lib.ptr(R), _lib.ptr(info))
    torch.cuda.synchronize()
    Gh = G.cpu().numpy()
    Rref, kept = _chol_drop_ref(Gh, 1e-6, shift)
    r = int(info[0].item())
    assert r == len(kept) == ell - len(dup)
    assert [j for j in range(ell) if j not in kept] == dup
    Rg = R.cpu().numpy()
    assert np.abs(Rg - Rref).max() <= 1e-9 * np.abs(Rref).max()
    Pg = P.cpu().numpy()
    Rk = Rref[np.ix_(kept, kept)]
    Pk = Pg[np.ix_(kept, np.arange(r))]
    assert np.abs(Rk @ Pk - np.eye(r)).max() <= 1e-8
    assert np.abs(np.delete(Pg, kept, axis=0)).max() == 0.0
    if r < ell:
        assert np.abs(Pg[:, r:]).max() == 0.0


def test_orth_ill_conditioned_panel():
    """kappa(Y) ~ 1e7 (cfg5-like): fp64 Gram CholQR2 cannot resolve it; the
    guarded fallback must still give the reference's Q."""
    from oracle import lowrank_oracle as O
    g = np.random.default_rng(5)
    U = np.linalg.qr(g.standard_normal((3000, 48)))[0]
    V = np.linalg.qr(g.standard_normal((48, 48)))[0]
    s = np.logspace(0, -7.5, 48)
    Y = (U * s) @ V.T
    Q = lr().orthonormalize_double_gs(Y)
    Qo = O.orthonormalize_double_gs(Y)
    assert Q.shape == Qo.shape
    assert np.linalg.norm(Q.T @ Q - np.eye(Q.shape[1])) <= 1e-12 * 48
    # span agreement: the projector difference is tiny where the oracle is accurate
    assert np.linalg.norm(Q @ (Q.T @ Qo) - Qo) <= 1e-6


def test_orth_golden_kats(golden):
    g = golden("kats")
    m = lr()
    Q = m.orthonormalize_double_gs(np.array([[1.0, 2.0], [0.0, 0.0]]))
    assert Q.shape == (2, 1) and np.allclose(Q, g["dgs_collinear"], atol=1e-14)
    Q = m.orthonormalize_double_gs(g["dgs_neardep_Y"])
    assert Q.shape == (100, 9)
    assert np.abs(Q - g["dgs_neardep_Q"]).max() <= 1e-10
    for key in ("dgs_rand", "dgs_cplx"):
        Q = m.orthonormalize_double_gs(g[f"{key}_Y"])
        assert np.abs(Q - g[f"{key}_Q"]).max() <= 1e-12
    assert m.orthonormalize_double_gs(np.zeros((5, 3))).shape == (5, 0)
    Q = m.orthonormalize_double_gs(np.eye(4))
    assert np.allclose(np.abs(Q), np.eye(4))


def test_orth_tol_zero_keeps_tiny_columns():
    Y = np.random.default_rng(1).standard_normal((50, 4))
    Y[:, 2] = Y[:, 0] + 1e-9 * Y[:, 2]
    Q = lr().orthonormalize_double_gs(Y, tol=0.0)
    assert Q.shape == (50, 4)
    Q = lr().orthonormalize_double_gs(Y, tol=1e-8)
    assert Q.shape == (50, 3)


def test_small_svd_golden(golden):
    g = golden("kats")
    m = lr()
    s = m.small_svd(np.array([[1.0, 1.0], [0.0, 1.0]])).sigma
    assert s[0] == pytest.approx(1.6180339887, abs=1e-9)
    assert s[1] == pytest.approx(0.6180339887, abs=1e-9)
    for key in ("svd_rand", "svd_cplx"):
        f = m.small_svd(g[f"{key}_B"])
        assert np.abs(f.sigma - g[f"{key}_s"]).max() <= 1e-13
        assert np.abs(f.U - g[f"{key}_U"]).max() <= 1e-11
        assert np.abs(f.V - g[f"{key}_V"]).max() <= 1e-11
    assert np.allclose(m.small_svd(np.diag([3.0, 1.0])).sigma, [3.0, 1.0])
    assert np.allclose(m.small_svd(np.array([[0.0, 1.0], [1.0, 0.0]])).sigma, [1.0, 1.0])


@pytest.mark.parametrize("r,c", [(30, 2048), (110, 8192), (10, 7), (7, 7), (120, 300)])
def test_small_svd_vs_oracle(r, c):
    from oracle import lowrank_oracle as O
    B = rand((r, c), np.float64, r * c)
    f = lr().small_svd(B)
    fo = O.small_svd(B)
    assert np.abs(f.sigma - fo.sigma).max() <= 1e-13 * fo.sigma[0]
    k = min(r, c)
    assert np.abs(f.U - fo.U).max() <= 1e-10
    assert np.abs(f.V - fo.V).max() <= 1e-10
    assert np.linalg.norm((f.U * f.sigma) @ f.V.T - B) <= 1e-13 * np.linalg.norm(B) * k


def test_small_svd_graded():
    """Graded spectrum down to 1e-8 (cfg5-like): relative accuracy of the
    small singular values through CholeskyQR + one-sided Jacobi."""
    from oracle import lowrank_oracle as O
    g = np.random.default_rng(3)
    U = np.linalg.qr(g.standard_normal((48, 48)))[0]
    V = np.linalg.qr(g.standard_normal((5000, 48)))[0]
    s = np.logspace(0, -8, 48)
    B = (U * s) @ V.T
    f = lr().small_svd(B)
    assert np.all(np.abs(f.sigma - s) <= 1e-8 * s + 1e-15)


def test_small_svd_rank_deficient():
    B = np.zeros((3, 6))
    B[0, 0] = 2.0
    f = lr().small_svd(B)
    assert np.allclose(f.sigma, [2.0, 0.0, 0.0])
    assert np.allclose((f.U * f.sigma) @ f.V.T, B, atol=1e-14)


def test_dft_and_srft_golden(golden):
    g = golden("kats")
    m = lr()
    assert np.allclose(m.dft(np.array([1.0, 0.0])), g["dft_n2"], atol=1e-15)
    assert np.allclose(m.dft(np.ones(4)), g["dft_n4"], atol=1e-15)
    assert np.abs(m.dft(g["dft16_in"], axis=1) - g["dft16_out"]).max() <= 1e-13
    Y = m.srft_apply(g["srft_A"], m.srft_operator(16, 4, 1))
    assert np.abs(Y - g["srft_Y"]).max() <= 1e-13
    # non-power-of-two length (the reference's Bluestein path)
    assert np.abs(m.dft(g["dft12_in"], axis=1) - g["dft12_out"]).max() <= 1e-13


@pytest.mark.parametrize("n", [64, 1024, 8192, 12, 1000, 6000])
def test_srft_vs_oracle(n):
    from oracle import lowrank_oracle as O
    A = rand((33, n), np.complex128, n)
    ell = min(17, n)
    op = O.srft_operator(n, ell, 9)
    Y = lr().srft_apply(A, lr().srft_operator(n, ell, 9))
    Yo = O.srft_apply(A, op)
    assert np.abs(Y - Yo).max() <= 1e-12 * np.abs(Yo).max()
    A32 = A.astype(np.complex64)
    Y32 = lr().srft_apply(A32, lr().srft_operator(n, ell, 9))
    assert np.abs(Y32 - Yo).max() <= 2e-5 * np.abs(Yo).max()


def test_gsrft_golden_and_oracle(golden):
    """Givens-chain SRFT (reference sketch.py:221-337) on the device: the
    reference's own outputs (power-of-two and not) and the oracle at size."""
    from oracle import lowrank_oracle as O
    g = golden("kats")
    m = lr()
    Y = m.gsrft_apply(g["gsrft_A"], m.gsrft_operator(16, 4, 2))
    assert np.abs(Y - g["gsrft_Y"]).max() <= 1e-12
    Y = m.gsrft_apply(g["gsrft12_A"], m.gsrft_operator(12, 5, 7))
    assert np.abs(Y - g["gsrft12_Y"]).max() <= 1e-12
    b = m.fast_range_finder(g["rf_A"][:, :16], 5, 4, kind="gsrft")
    assert np.abs(b.Q - g["rf_gsrft_Q"]).max() <= 1e-10
    for n, dt, tol in [(1024, np.complex128, 1e-11), (1000, np.complex128, 1e-11),
                       (2048, np.complex64, 2e-5)]:
        A = rand((300, n), dt, n + 1)
        Yd = m.gsrft_apply(A, m.gsrft_operator(n, 40, 3))
        Yo = O.gsrft_apply(A.astype(np.complex128), O.gsrft_operator(n, 40, 3))
        assert np.abs(Yd - Yo).max() <= tol * np.abs(Yo).max()


@pytest.mark.parametrize("mode", ["", "warp", "half", "slice4", "slice8"])
@pytest.mark.parametrize("ell", [1, 5, 16, 17, 33, 48, 64, 65, 100])
def test_csr_spmm_vs_scipy(ell, mode, monkeypatch):
    """Every SpMM kernel (row-major gathers, and the L2-resident column
    slices that config 5 takes) on ragged, dense and empty rows."""
    import scipy.sparse as sp
    from paper_0909_4061_b200.sparse import CudaCsrOperator
    if mode:
        monkeypatch.setenv("LR_SPMM", mode)
    g = np.random.default_rng(4)
    S = sp.random(3000, 2500, density=0.004, random_state=4, format="csr").tolil()
    S[7, :] = g.standard_normal(2500)        # a dense row: many 32-nonzero chunks
    S[11, :70] = 1.0                         # a ragged row (70 = 2*32 + 6)
    S[13, :] = 0.0                           # an empty row
    S = S.tocsr()
    L = g.standard_normal((3000, 5))
    R = g.standard_normal((2500, 5))
    op = CudaCsrOperator(S, L, R)
    X = g.standard_normal((2500, ell))
    Y = g.standard_normal((3000, ell))
    assert np.abs(op.apply(X) - (S @ X + L @ (R.T @ X))).max() <= 1e-12 * 500
    assert np.abs(op.apply_adjoint(Y) - (S.T @ Y + R @ (L.T @ Y))).max() <= 1e-12 * 500
    op2 = CudaCsrOperator(S)
    assert np.abs(op2.apply(X) - S @ X).max() <= 1e-11


def test_estimate_matches_oracle():
    from oracle import lowrank_oracle as O
    A = rand((400, 300), np.float64, 7)
    Q = np.linalg.qr(rand((400, 20), np.float64, 8))[0]
    e = lr().posterior_error_estimate(A, Q, r=10, alpha=10.0, seed=5)
    eo = O.posterior_error_estimate(A, Q, r=10, alpha=10.0, seed=5)
    assert e == pytest.approx(eo, rel=1e-12)
    assert lr().posterior_error_estimate(A, np.zeros((400, 0)), seed=5) == pytest.approx(
        O.posterior_error_estimate(A, np.zeros((400, 0)), seed=5), rel=1e-12)


@pytest.mark.parametrize("seed,stream,n,ell", [(2, 0x67617573, 8192, 110), (1, 0x67617573, 2048, 30),
                                               (15, 0x70726F62, 8192, 10), (4, 0x67617573, 4096, 256),
                                               (123456789, 0x67617573, 1 << 16, 48)])
def test_device_gaussian_matches_numpy_stream(seed, stream, n, ell):
    """K0: the device Philox/ziggurat stream equals numpy's (reference
    sketch.py:32-42,96-100) -- all but at most the last ulp of tail draws."""
    from paper_0909_4061_b200.sketch import gaussian_dev, rng_for
    ref = rng_for(seed, stream).standard_normal((n, ell))
    got = gaussian_dev(n, ell, seed, stream=stream).cpu().numpy()
    diff = np.flatnonzero(ref != got)
    assert diff.size <= max(2, ref.size // 200000)
    if diff.size:
        assert np.all(np.abs(ref.ravel()[diff]) > 3.654)
        assert np.abs(ref.ravel()[diff] - got.ravel()[diff]).max() <= 4e-15 * np.abs(ref).max()
    g32 = gaussian_dev(n, ell, seed, stream=stream, dtype=torch.float32).cpu().numpy()
    assert (g32 != ref.astype(np.float32)).sum() <= diff.size


@pytest.mark.parametrize("dtype", [np.float64, np.complex128, np.float32])
def test_passes_deterministic(dtype):
    """Repeated identical range finders give bitwise-identical bases: the
    TMA-fed pass kernels release a stage to the TMA engine only after the
    consumers' shared loads are ordered before the refill (a missing proxy
    fence once let refills land under in-flight loads: ~1e-2 run-to-run
    differences in Q, tools/flaky_eig.py)."""
    m = lr()
    g = np.random.default_rng(21)
    A = rand((3000, 2500), dtype, 21)
    Qs = [m.randomized_range_finder(A, 40, seed=3).Q for _ in range(6)]
    for Q in Qs[1:]:
        assert np.array_equal(Q, Qs[0])


@pytest.mark.parametrize("M,N,K", [(32, 48, 2 ** 18), (48, 48, 20000), (10, 30, 16384),
                                   (30, 30, 70001), (32, 64, 40000), (1, 1, 16384)])
def test_skinny_tn(M, N, K):
    """A^T B with K >> M, N (the Grams of narrow panels and config 5's R^T X):
    the skinny kernel against numpy, and symmetric when A is B."""
    from paper_0909_4061_b200 import _lib
    g = np.random.default_rng(M * N + K)
    A = torch.from_numpy(g.standard_normal((K, M))).cuda()
    B = torch.from_numpy(g.standard_normal((K, N))).cuda()
    C = torch.empty((M, N), dtype=torch.float64, device="cuda")
    _lib.call("lr_gemm", _lib.handle(), _lib.F64, _lib.OP_T, K, M, N, _lib.ptr(A), _lib.ld(A),
              _lib.ptr(B), _lib.ld(B), _lib.ptr(C), _lib.ld(C))
    ref = A.cpu().numpy().T @ B.cpu().numpy()
    assert np.abs(C.cpu().numpy() - ref).max() <= 1e-12 * np.sqrt(K) * 4
    G = torch.empty((M, M), dtype=torch.float64, device="cuda")
    _lib.call("lr_gemm", _lib.handle(), _lib.F64, _lib.OP_T, K, M, M, _lib.ptr(A), _lib.ld(A),
              _lib.ptr(A), _lib.ld(A), _lib.ptr(G), _lib.ld(G))
    Gh = G.cpu().numpy()
    assert np.array_equal(Gh, Gh.T) or np.abs(Gh - Gh.T).max() <= 1e-12 * np.abs(Gh).max()
    assert np.abs(Gh - A.cpu().numpy().T @ A.cpu().numpy()).max() <= 1e-12 * np.sqrt(K) * 4


@pytest.mark.parametrize("M,N,K", [(2 ** 18, 48, 32), (100003, 48, 48), (70000, 30, 30),
                                   (65536, 64, 32), (65537, 1, 1), (131072, 10, 20)])
def test_skinny_nn(M, N, K):
    """A B with M >> K, N (the applies Y P of narrow panels, config 5's L Z):
    the skinny NN kernel against numpy, including ragged last tiles."""
    from paper_0909_4061_b200 import _lib
    g = np.random.default_rng(M + N + K)
    A = torch.from_numpy(g.standard_normal((M, K))).cuda()
    B = torch.from_numpy(g.standard_normal((K, N))).cuda()
    C = torch.empty((M, N + (N % 2)), dtype=torch.float64, device="cuda")[:, :N]
    _lib.call("lr_gemm", _lib.handle(), _lib.F64, _lib.OP_N, M, K, N, _lib.ptr(A), _lib.ld(A),
              _lib.ptr(B), _lib.ld(B), _lib.ptr(C), _lib.ld(C))
    ref = A.cpu().numpy() @ B.cpu().numpy()
    assert np.abs(C.cpu().numpy() - ref).max() <= 1e-13 * K


@pytest.mark.parametrize("m,n,ell", [(300, 257, 30), (129, 64, 110), (2048, 2048, 30),
                                     (1000, 3000, 64), (513, 77, 128), (4096, 700, 200),
                                     (37, 1, 3), (5000, 40, 7)])
@pytest.mark.parametrize("adjoint", [False, True])
def test_ozaki_fp64_pass(m, n, ell, adjoint):
    """fp64 passes on the int8 tensor cores (lr_gemm_ozaki): every entry
    within 2^-50 of the |A||X| bound of an fp64 GEMM (the reference's
    OpenBLAS dgemm has the same bound), checked against an 80-bit product;
    deterministic bit for bit."""
    from paper_0909_4061_b200 import core
    g = np.random.default_rng(m + n + ell)
    A = g.standard_normal((m, n)) * np.exp(g.uniform(-3, 3, (m, 1)))   # rows of mixed scale
    X = g.standard_normal((m if adjoint else n, ell)) * np.exp(g.uniform(-3, 3, (1, ell)))
    Ad, Xd = torch.from_numpy(A).cuda(), torch.from_numpy(X).cuda()
    oz = core.ozaki_prepare(Ad)
    rows = n if adjoint else m
    Y = torch.empty((rows, ell), dtype=torch.float64, device="cuda")
    core.ozaki_pass(oz, m, n, Xd, Y, adjoint)
    Y2 = torch.empty_like(Y)
    core.ozaki_pass(oz, m, n, Xd, Y2, adjoint)
    assert torch.equal(Y, Y2)
    Al, Xl = A.astype(np.longdouble), X.astype(np.longdouble)
    ref = (Al.T @ Xl) if adjoint else (Al @ Xl)
    bound = (np.abs(A).T @ np.abs(X)) if adjoint else (np.abs(A) @ np.abs(X))
    err = np.abs(Y.cpu().numpy().astype(np.longdouble) - ref)
    assert float((err / np.maximum(bound, 1e-300)).max()) <= 2.0 ** -50


@pytest.mark.parametrize("M,N,K", [(256, 256, 256), (110, 110, 110), (30, 30, 30), (16, 500, 33),
                                   (257, 19, 512), (120, 240, 240), (48, 48, 1)])
@pytest.mark.parametrize("trans", [False, True])
def test_gemm_small(M, N, K, trans):
    """fp64 products small in every dimension (gemm_small.cu: one 32 x 32 tile
    per CTA, no split-K) -- the ell^3 algebra around the factorizations --
    against numpy, both operand orientations, ragged tiles, and a strided C."""
    from paper_0909_4061_b200 import _lib
    g = np.random.default_rng(M + 7 * N + 13 * K)
    A = torch.from_numpy(g.standard_normal((K, M) if trans else (M, K))).cuda()
    B = torch.from_numpy(g.standard_normal((K, N))).cuda()
    Cfull = torch.zeros((M, N + 3), dtype=torch.float64, device="cuda")
    C = Cfull[:, :N]
    rows, cols = A.shape
    _lib.call("lr_gemm", _lib.handle(), _lib.F64, _lib.OP_T if trans else _lib.OP_N, rows, cols, N,
              _lib.ptr(A), _lib.ld(A), _lib.ptr(B), _lib.ld(B), _lib.ptr(C), _lib.ld(C))
    An = A.cpu().numpy()
    ref = (An.T if trans else An) @ B.cpu().numpy()
    assert np.abs(C.cpu().numpy() - ref).max() <= 1e-14 * max(K, 16) * 4
    assert float(Cfull[:, N:].abs().max()) == 0.0        # nothing written past N


def test_csr_transpose_on_device_is_canonical():
    """The CSR of S^T built on the device (stable sort by column) equals
    scipy's canonical transpose: same row pointers, indices ascending in every
    row, same values -- including empty rows / columns and merged duplicates."""
    import scipy.sparse as sp
    from paper_0909_4061_b200.sparse import CudaCsrOperator
    g = np.random.default_rng(12)
    rows = g.integers(0, 900, 6000)
    cols = g.integers(0, 700, 6000)
    cols[cols == 5] = 6                      # an empty column
    rows[rows == 17] = 18                    # an empty row
    vals = g.standard_normal(6000)
    S = sp.coo_matrix((vals, (rows, cols)), shape=(900, 700)).tocsr()   # duplicates are summed
    op = CudaCsrOperator(S)
    St = S.T.tocsr()
    St.sum_duplicates()
    St.sort_indices()
    ptr, idx, val = (t.cpu().numpy() for t in op.St)
    assert np.array_equal(ptr, St.indptr.astype(np.int64))
    assert np.array_equal(idx, St.indices.astype(np.int32))
    assert np.array_equal(val, St.data)


@pytest.mark.parametrize("M,N,K", [(8192, 110, 110), (16384, 110, 110), (5000, 65, 128), (4099, 128, 9),
                                   (70000, 96, 96), (4096, 127, 101)])
def test_skinny_nn_wide(M, N, K):
    """A B with 64 < N <= 128, K <= 128 and a tall A (config 2's ell = 110 panel
    applies): the wide skinny kernel against numpy, ragged tiles and odd K; and
    through the orthonormalization, whose triangular factor skips k-blocks."""
    from paper_0909_4061_b200 import _lib, core
    g = np.random.default_rng(M + N + K)
    A = torch.from_numpy(g.standard_normal((M, K))).cuda()
    B = torch.from_numpy(g.standard_normal((K, N))).cuda()
    C = torch.empty((M, N + (N % 2)), dtype=torch.float64, device="cuda")[:, :N]
    _lib.call("lr_gemm", _lib.handle(), _lib.F64, _lib.OP_N, M, K, N, _lib.ptr(A), _lib.ld(A),
              _lib.ptr(B), _lib.ld(B), _lib.ptr(C), _lib.ld(C))
    ref = A.cpu().numpy() @ B.cpu().numpy()
    assert np.abs(C.cpu().numpy() - ref).max() <= 1e-13 * K
    if N == K:
        Y = (A * torch.logspace(0, -4, K, device="cuda", dtype=torch.float64)) @ B
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        with core.speculate(status):
            Q = core.orth_dev(Y)
        torch.cuda.synchronize()
        assert int(status.item()) == 0
        Qn, Yn = Q.cpu().numpy(), Y.cpu().numpy()
        assert np.abs(Qn.T @ Qn - np.eye(N)).max() <= 1e-13
        Rm = Qn.T @ Yn
        assert np.linalg.norm(np.tril(Rm, -1)) <= 1e-12 * np.linalg.norm(Rm)
        assert np.linalg.norm(Yn - Qn @ Rm) <= 1e-13 * np.linalg.norm(Yn)
