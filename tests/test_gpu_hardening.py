"""Robustness of the fast paths against their failure modes (VERDICT r1
"What's weak" #2/#3): in-place changes of A between CUDA-graph
replays, scratch-pool chunks freed under a captured graph, and fp64 rows
whose entries span many decades (the int8 digit planes are fixed-point per
row)."""

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


def _spectrum_matrix(rows, cols, seed, dtype):
    g = np.random.default_rng(seed)
    A = g.standard_normal((rows, cols)) * (np.arange(1, cols + 1) ** -0.5)
    return torch.from_numpy(A.astype(dtype)).cuda()


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_graph_replay_follows_inplace_update(dtype, monkeypatch):
    """After the step of an operator is captured and replayed, A.mul_(2)
    must double sigma on the next call (the int8 digit planes / max|A| of
    the old A must not be replayed)."""
    m = lr()
    monkeypatch.setenv("LR_OZAKI", "1")
    Ad = _spectrum_matrix(3000, 1500, 5, dtype)
    op = m.DenseOperator(Ad)
    outs = [m.randomized_svd(op, 40, 10, 1, 3, estimate=False)[1].sigma.clone()
            for _ in range(4)]          # eager, eager + capture, replay, replay
    for s in outs[1:]:
        assert torch.equal(s, outs[0])
    Ad.mul_(2.0)
    s2 = m.randomized_svd(op, 40, 10, 1, 3, estimate=False)[1].sigma
    fresh = m.randomized_svd(m.DenseOperator(Ad.clone()), 40, 10, 1, 3,
                             estimate=False)[1].sigma
    tol = 1e-12 if dtype == "float64" else 1e-5
    assert torch.allclose(s2, 2.0 * outs[0], rtol=tol, atol=0)
    assert torch.allclose(s2, fresh, rtol=tol, atol=0)
    if dtype == "float32":
        assert op.amax == pytest.approx(float(Ad.abs().max()), rel=0)


def test_pool_merge_invalidates_captured_graph():
    """A call that outgrows the handle's scratch pool makes the next call
    merge (free) the chunks; a graph captured before must then not be
    replayed (lr_pool_generation), and the step still gives the same
    factors."""
    m = lr()
    from paper_0909_4061_b200 import _lib
    Ad = _spectrum_matrix(2000, 800, 7, "float64")
    op = m.DenseOperator(Ad)
    ref = [m.randomized_svd(op, 30, 10, 1, 2, estimate=False)[1] for _ in range(3)][-1]
    h = _lib.handle()
    gen0 = _lib.pool_generation(h)
    big = _spectrum_matrix(40000, 2048, 8, "float64")
    m.randomized_svd(big, 200, 40, 1, 2, estimate=False)     # grows the pool
    del big
    m.randomized_svd(op, 30, 10, 1, 2, estimate=False)        # merge happens here
    assert _lib.pool_generation(h) > gen0
    f = m.randomized_svd(op, 30, 10, 1, 2, estimate=False)[1]
    assert torch.equal(f.sigma, ref.sigma)
    assert torch.equal(f.U, ref.U)
    torch.cuda.synchronize()


def test_ozaki_row_scale_bound():
    """Rows graded over 6 decades (not flagged: only isolated Gaussian tiny
    entries fall below 2^-32 of the row maximum): the int8 pass meets
    its stated bound |err_ij| <= 2^-50 max_k|A_ik| sum_k|X_kj| against an
    80-bit product (A X), and the normwise bound for A^T Y."""
    from paper_0909_4061_b200 import core
    g = np.random.default_rng(31)
    m_, n_, ell = 700, 1024, 48
    A = g.standard_normal((m_, n_)) * np.logspace(0, -6, n_)
    A[5, 7] = 1e-30                      # an isolated tiny entry does not flag the row
    X = g.standard_normal((n_, ell))
    Ad = torch.from_numpy(A).cuda()
    oz = core.ozaki_prepare(Ad)
    assert int(oz[3].item()) == 0
    Y = torch.empty((m_, ell), dtype=torch.float64, device="cuda")
    core.ozaki_pass(oz, m_, n_, torch.from_numpy(X).cuda(), Y, False)
    ref = A.astype(np.longdouble) @ X.astype(np.longdouble)
    err = np.abs(Y.cpu().numpy().astype(np.longdouble) - ref)
    bound = np.abs(A).max(axis=1, keepdims=True) * np.abs(X).sum(axis=0, keepdims=True)
    assert float((err / bound).max()) <= 2.0 ** -50
    Yt = g.standard_normal((m_, ell))
    Z = torch.empty((n_, ell), dtype=torch.float64, device="cuda")
    core.ozaki_pass(oz, m_, n_, torch.from_numpy(Yt).cuda(), Z, True)
    reft = A.T.astype(np.longdouble) @ Yt.astype(np.longdouble)
    errt = np.abs(Z.cpu().numpy().astype(np.longdouble) - reft)
    rmax = np.abs(A).max(axis=1, keepdims=True)
    bound_t = (rmax * np.abs(Yt)).max(axis=0, keepdims=True) * m_
    assert float((errt / bound_t).max()) <= 2.0 ** -50


def test_ozaki_wide_rows_fall_back_to_dmma(monkeypatch):
    """Graded rows spanning 12 decades (a quarter of each row below 2^-32 of
    its maximum): lr_ozaki_prepare flags them and the passes stay on DMMA,
    whose error is relative to |A||X| entrywise."""
    m = lr()
    from paper_0909_4061_b200 import core
    monkeypatch.setenv("LR_OZAKI", "auto")
    g = np.random.default_rng(32)
    m_, n_, ell = 2048, 1024, 64
    A = g.standard_normal((m_, n_)) * np.logspace(0, -12, n_)
    Ad = torch.from_numpy(A).cuda()
    oz = core.ozaki_prepare(Ad)
    assert int(oz[3].item()) == m_
    assert core._ozaki_planes(Ad) is None
    X = np.zeros((n_, ell))
    X[n_ // 2:] = g.standard_normal((n_ - n_ // 2, ell))   # weight on the small columns
    op = m.DenseOperator(Ad)
    Y = op.apply(torch.from_numpy(X).cuda()).cpu().numpy()
    ref = A.astype(np.longdouble) @ X.astype(np.longdouble)
    bound = np.abs(A) @ np.abs(X)
    err = np.abs(Y.astype(np.longdouble) - ref)
    assert float((err / bound).max()) <= 2.0 ** -44


# ---- sketch-preconditioned CholeskyQR of tall fp32 panels (sketch_rows.cu) ----------

def _tall_panel(m, ell, kappa, seed, heavy_rows=False):
    g = torch.Generator(device="cuda").manual_seed(seed)
    U = torch.randn(m, ell, device="cuda", dtype=torch.float64, generator=g)
    if heavy_rows:
        U[:: m // 64] *= 300.0
    U, _ = torch.linalg.qr(U)
    W, _ = torch.linalg.qr(torch.randn(ell, ell, device="cuda", dtype=torch.float64, generator=g))
    s = torch.logspace(0, -float(np.log10(kappa)), ell, device="cuda", dtype=torch.float64)
    return ((U * s) @ W.T).float().contiguous()


def _orth_quality(Y, Q):
    Qd, Yd = Q.double(), Y.double()
    ell = Q.shape[1]
    orth = (Qd.T @ Qd - torch.eye(ell, device="cuda", dtype=torch.float64)).abs().max().item()
    R = Qd.T @ Yd
    span = (torch.linalg.norm(Yd - Qd @ R) / torch.linalg.norm(Yd)).item()
    low = (torch.linalg.norm(torch.tril(R, -1)) / torch.linalg.norm(R)).item()
    return orth, span, low


@pytest.mark.parametrize("m,ell,kappa,heavy", [(131072, 256, 1e6, False), (262144, 128, 1e3, False),
                                               (131072, 256, 1e6, True), (100003, 72, 1e4, False)])
def test_sketch_preconditioned_orth(m, ell, kappa, heavy):
    """Tall fp32 panels take the sketch-preconditioned CholeskyQR (no exact
    Gram): the speculative step must report no flag and return the
    Gram-Schmidt basis of Y -- orthonormal at the fp32 rounding level, the
    same span, Q^T Y upper triangular (reference core.py:84-115 builds the
    columns in order).  Heavy rows are the hard case for a sparse embedding."""
    from paper_0909_4061_b200 import core
    Y = _tall_panel(m, ell, kappa, 11, heavy)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    with core.speculate(status):
        Q = core.orth_dev(Y)
        Q1, P2 = core.orth_dev_deferred(Y)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    orth, span, low = _orth_quality(Y, Q)
    assert orth <= (2e-5 if heavy else 1e-6), orth
    assert span <= (3e-5 if heavy else 5e-6), span
    assert low <= (2e-5 if heavy else 2e-6), low
    # the deferred pair spans the same space (range only: its Q1 P2 is
    # orthonormal to the tensor-core Gram's ~2e-5)
    Qd = (Q1.double() @ P2)
    assert (Qd.T @ Qd - torch.eye(ell, device="cuda", dtype=torch.float64)).abs().max().item() <= 2e-4
    Yd = Y.double()
    Qo, _ = torch.linalg.qr(Qd)
    assert (torch.linalg.norm(Yd - Qo @ (Qo.T @ Yd)) / torch.linalg.norm(Yd)).item() <= (3e-5 if heavy else 5e-6)


def test_sketch_preconditioned_orth_flags_rank_deficiency():
    """A dependent column must not be decided from the sketch: the speculative
    step flags it and the exact path drops it like the reference."""
    from paper_0909_4061_b200 import core
    Y = _tall_panel(131072, 64, 10.0, 5)
    Y[:, 40] = Y[:, 3] * 0.5     # exactly dependent in fp32 too
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    with core.speculate(status):
        core.orth_dev(Y)
    torch.cuda.synchronize()
    assert int(status.item()) & 3        # dropped or unresolved pivot: exact path
    Q = core.orth_dev(Y)
    assert Q.shape[1] == 63
    orth, span, _ = _orth_quality(Y, Q)
    assert orth <= 1e-6 and span <= 5e-6


def test_sketch_preconditioned_orth_repeatable():
    """Bitwise run-to-run determinism (fixed-order partial sums, no atomics on data)."""
    from paper_0909_4061_b200 import core
    Y = _tall_panel(131072, 128, 1e5, 9)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    outs = []
    for _ in range(2):
        with core.speculate(status):
            outs.append(core.orth_dev(Y).clone())
    assert torch.equal(outs[0], outs[1])


def test_sketch_preconditioned_orth_strided_panel():
    """The panel may be a column slice of a wider array (row stride > ell)."""
    from paper_0909_4061_b200 import core
    wide = _tall_panel(131072, 256, 1e5, 21)
    Y = wide[:, 64:192]
    assert Y.stride(0) == 256 and Y.shape[1] == 128
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    with core.speculate(status):
        Q = core.orth_dev(Y)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    orth, span, low = _orth_quality(Y.contiguous(), Q)
    assert orth <= 1e-6 and span <= 5e-6 and low <= 2e-6
