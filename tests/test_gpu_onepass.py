"""One-pass sketches, the LRKMAT00 reader and row-block streaming on the GPU
 against the reference's own outputs
(tests/golden/onepass.npz, made by tests/golden/make_golden.py from
/root/reference) and the reference's tests (tests/test_io.py:160-209,
tests/test_factor.py:253-314)."""

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


def test_svd_one_pass_general_vs_reference(golden):
    from paper_0909_4061_b200 import factor
    g = golden("onepass")
    b = factor.sample_bundle_two_sided(g["gen_A"], 15, seed=6)
    assert b.Q.shape == g["gen_Q"].shape and b.Q_tilde.shape == g["gen_Qt"].shape
    assert np.abs(b.Y - g["gen_Y"]).max() <= 1e-12 * np.abs(g["gen_Y"]).max()
    f = factor.svd_one_pass_general(b)
    assert np.abs(f.sigma - g["gen_sigma"]).max() <= 1e-10 * g["gen_sigma"][0]
    assert np.abs(f.compose() - g["gen_comp"]).max() <= 1e-9 * np.abs(g["gen_comp"]).max()
    for tag, rank in (("gen2", None), ("gen2r", 10)):
        b = factor.sample_bundle_two_sided(g["gen2_A"], 20, ell_tilde=24, seed=9, rank=rank)
        f = factor.svd_one_pass_general(b)
        ref = g[f"{tag}_sigma"]
        assert np.abs(f.sigma - ref).max() <= 1e-10 * ref[0]
        assert np.abs(f.compose() - g[f"{tag}_comp"]).max() <= 1e-9 * np.abs(g[f"{tag}_comp"]).max()


def test_eig_one_pass_vs_reference(golden):
    from paper_0909_4061_b200 import factor
    g = golden("onepass")
    for tag, ell, rank in (("herm", 16, None), ("herm2", 20, 10)):
        b = factor.sample_bundle(g[f"{tag}_H"], ell, seed=5, rank=rank)
        assert b.q_choice == ("gs" if rank is None else "svd")
        e = factor.eig_one_pass(b)
        lam = g[f"{tag}_lam"]
        assert np.abs(e.lam - lam).max() <= 1e-9 * np.abs(lam).max()
        assert e.diagnostics["tau_min"] == pytest.approx(g[f"{tag}_tau"][0], rel=1e-9)
        assert np.abs(e.compose() - g[f"{tag}_comp"]).max() <= 1e-8 * np.abs(lam).max()


def test_one_pass_contracts():
    """Reference tests/test_factor.py:275-314: zero bundles, dimension cap."""
    from paper_0909_4061_b200 import config, factor
    b = factor.sample_bundle(np.zeros((8, 8)), 3, seed=0)
    assert np.allclose(factor.eig_one_pass(b).lam, 0.0)
    b = factor.sample_bundle_two_sided(np.zeros((6, 5)), 3, seed=0)
    f = factor.svd_one_pass_general(b)
    assert f.sigma.size == 0 or np.allclose(f.sigma, 0.0)
    old = config.ONE_PASS_DIM_CAP
    config.ONE_PASS_DIM_CAP = 4
    try:
        A = np.random.default_rng(22).standard_normal((20, 20))
        with pytest.raises(ValueError, match="two-pass"):
            factor.svd_one_pass_general(factor.sample_bundle_two_sided(A, 6, seed=3))
    finally:
        config.ONE_PASS_DIM_CAP = old


@pytest.mark.parametrize("tag,br,ell", [("st", 8, 6), ("stc", 5, 4)])
def test_streamed_bundle_vs_reference(golden, tmp_path, tag, br, ell):
    """The LRKMAT00 writer is byte-identical; the streamed two-sided bundle
    (device blocks through pinned buffers) matches the reference's, equals
    the in-memory bundle with the same block size bitwise, and repeats
    bitwise."""
    from paper_0909_4061_b200 import io as lio
    g = golden("onepass")
    A = g[f"{tag}_A"]
    p = tmp_path / f"{tag}.bin"
    lio.write_matrix_binary(A, p)
    assert np.array_equal(np.frombuffer(p.read_bytes()[:64], dtype=np.uint8), g[f"{tag}_bytes"])
    sb = lio.streamed_sample_bundle(lio.stream_row_blocks(p, br), ell=ell, seed=4)
    assert np.abs(sb.Omega - g[f"{tag}_Om"]).max() <= 4e-16 * np.abs(g[f"{tag}_Om"]).max()
    assert np.abs(sb.Omega_tilde - g[f"{tag}_Omt"]).max() <= 4e-16 * np.abs(g[f"{tag}_Omt"]).max()
    scale = np.abs(A).max() * A.shape[1]
    assert np.abs(sb.Y - g[f"{tag}_Y"]).max() <= 1e-13 * scale
    assert np.abs(sb.Y_tilde - g[f"{tag}_Yt"]).max() <= 1e-13 * np.abs(A).max() * A.shape[0]
    assert np.abs(sb.Q - g[f"{tag}_Q"]).max() <= 1e-10
    im = lio.in_memory_sample_bundle(A, ell=ell, seed=4, block_rows=br)
    assert np.array_equal(im.Y, sb.Y) and np.array_equal(im.Y_tilde, sb.Y_tilde)
    sb2 = lio.streamed_sample_bundle(lio.stream_row_blocks(p, br), ell=ell, seed=4)
    assert np.array_equal(sb2.Y, sb.Y) and np.array_equal(sb2.Y_tilde, sb.Y_tilde)
    host = lio.streamed_sample_bundle(lio.stream_row_blocks(p, br), ell=ell, seed=4,
                                      device_blocks=False)
    assert np.array_equal(host.Y, sb.Y) and np.array_equal(host.Y_tilde, sb.Y_tilde)


def test_reader_errors_and_device_read(tmp_path):
    """Reference tests/test_io.py:95-110,160-185: bad magic, truncation,
    block row accounting; the device reader returns the same matrix."""
    from paper_0909_4061_b200 import io as lio
    rng = np.random.default_rng(8)
    A = rng.standard_normal((17, 4))
    p = tmp_path / "m.bin"
    lio.write_matrix_binary(A, p)
    blocks = list(lio.stream_row_blocks(p, 5))
    assert [r for r, _ in blocks] == [0, 5, 10, 15]
    assert sum(b.shape[0] for _, b in blocks) == 17
    assert np.array_equal(lio.read_matrix_binary(p), A)
    d = lio.read_matrix_binary(p, device="cuda")
    assert d.is_cuda and np.array_equal(d.cpu().numpy(), A)
    dev_blocks = [(r, b.cpu().numpy()) for r, b in lio.stream_row_blocks(p, 5).device_blocks()]
    assert [r for r, _ in dev_blocks] == [0, 5, 10, 15]
    assert np.array_equal(np.vstack([b for _, b in dev_blocks]), A)
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTMAGIC" + p.read_bytes()[8:])
    with pytest.raises(lio.MatrixFormatError):
        lio.read_matrix_binary(bad)
    trunc = tmp_path / "t.bin"
    trunc.write_bytes(p.read_bytes()[:-8 * 4])
    with pytest.raises(lio.StreamError):
        list(lio.stream_row_blocks(trunc, 4))
    with pytest.raises(lio.StreamError):
        list(lio.stream_row_blocks(trunc, 4).device_blocks())
    with pytest.raises(lio.MatrixFormatError):
        lio.read_matrix_binary(trunc)
    with pytest.raises(lio.MatrixFormatError):
        lio.read_matrix_binary(trunc, device="cuda")


def test_streamed_large_blocks_device_accumulation(tmp_path):
    """A 2^17 x 512 matrix streamed in 10000-row blocks (uneven last block):
    Y = A Omega and Y~ = A^T Omega~ agree with fp64 products of the same A
    and the reference's Omega draws to fp64 roundoff."""
    from oracle import lowrank_oracle as O
    from paper_0909_4061_b200 import io as lio
    rng = np.random.default_rng(31)
    m, n = 1 << 17, 512
    A = rng.standard_normal((m, n))
    p = tmp_path / "big.bin"
    lio.write_matrix_binary(A, p)
    sb = lio.streamed_sample_bundle(lio.stream_row_blocks(p, 10000), ell=24, ell_tilde=20, seed=7)
    Om, Omt = O.gaussian_matrix(n, 24, 7), O.gaussian_matrix(m, 20, 8)
    # the device generator matches numpy's stream to the last ulp on rare
    # ziggurat tail draws (tests/test_gpu_kernels.py)
    assert np.abs(sb.Omega - Om).max() <= 4e-16 * np.abs(Om).max()
    assert np.abs(sb.Omega_tilde - Omt).max() <= 4e-16 * np.abs(Omt).max()
    assert np.abs(sb.Y - A @ Om).max() <= 1e-12 * n
    assert np.abs(sb.Y_tilde - A.T @ Omt).max() <= 1e-12 * m
