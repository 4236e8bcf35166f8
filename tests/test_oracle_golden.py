"""Pin the CPU oracle (oracle/lowrank_oracle.py) to vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import workloads
from oracle import lowrank_oracle as O


def test_philox_draws_bitwise(golden):
    g = golden("kats")
    assert np.array_equal(O.gaussian_matrix(7, 3, 11), g["gauss_7x3_s11"])
    assert np.array_equal(O.probe_matrix(6, 2, 5), g["probe_6x2_s5"])
    d = O.srft_operator(64, 8, 3)
    assert np.array_equal(d.d, g["srft64_d"]) and np.array_equal(d.picks, g["srft64_picks"])
    d = O.srft_operator(8192, 120, 3)
    assert np.array_equal(d.d[:64], g["srft8192_d_head"])
    assert np.array_equal(d.picks, g["srft8192_picks"])
    assert np.allclose(d.d.sum(), g["srft8192_d_sum"][0], rtol=0, atol=1e-9)


def test_dgs_kats(golden):
    g = golden("kats")
    assert np.allclose(O.orthonormalize_double_gs(np.array([[1.0, 2.0], [0.0, 0.0]])),
                       g["dgs_collinear"])
    Q = O.orthonormalize_double_gs(g["dgs_neardep_Y"])
    assert Q.shape == g["dgs_neardep_Q"].shape == (100, 9)
    assert np.abs(Q - g["dgs_neardep_Q"]).max() <= 1e-13
    for key in ("dgs_rand", "dgs_cplx"):
        Q = O.orthonormalize_double_gs(g[f"{key}_Y"])
        assert np.abs(Q - g[f"{key}_Q"]).max() <= 1e-13
    assert O.orthonormalize_double_gs(np.zeros((5, 3))).shape == (5, 0)


def test_small_svd_kats(golden):
    g = golden("kats")
    s = O.small_svd(np.array([[1.0, 1.0], [0.0, 1.0]])).sigma
    assert np.allclose(s, g["svd_golden_s"], rtol=0, atol=1e-14)
    assert s[0] == pytest.approx(1.6180339887, abs=1e-9)
    for key in ("svd_rand", "svd_cplx"):
        f = O.small_svd(g[f"{key}_B"])
        assert np.abs(f.sigma - g[f"{key}_s"]).max() <= 1e-13
        assert np.abs(f.U - g[f"{key}_U"]).max() <= 1e-12
        assert np.abs(f.V - g[f"{key}_V"]).max() <= 1e-12


def test_dft_srft_kats(golden):
    g = golden("kats")
    assert np.allclose(O.dft(np.array([1.0, 0.0])), g["dft_n2"])
    assert np.allclose(O.dft(np.ones(4)), g["dft_n4"])
    assert np.abs(O.dft(g["dft16_in"], axis=1) - g["dft16_out"]).max() <= 1e-13
    assert np.abs(O.dft(g["dft12_in"], axis=1) - g["dft12_out"]).max() <= 1e-12
    Y = O.srft_apply(g["srft_A"], O.srft_operator(16, 4, 1))
    assert np.abs(Y - g["srft_Y"]).max() <= 1e-13


def test_range_finders_small(golden):
    g = golden("kats")
    A = g["rf_A"]
    assert np.abs(O.randomized_range_finder(A, 6, 11).Q - g["rf_basic_Q"]).max() <= 1e-12
    assert np.abs(O.power_iteration_range(A, 6, 2, 11).Q - g["rf_power_Q"]).max() <= 1e-10
    b = O.subspace_iteration_range(A, 6, 2, 11)
    assert np.abs(b.Q - g["rf_subspace_Q"]).max() <= 1e-12
    f = O.direct_svd(A, b.Q)
    assert np.abs(f.sigma - g["rf_dsvd_s"]).max() <= 1e-12
    assert np.abs(f.U - g["rf_dsvd_U"]).max() <= 1e-12
    assert np.abs(f.V - g["rf_dsvd_V"]).max() <= 1e-12
    assert O.posterior_error_estimate(A, b.Q, seed=3) == pytest.approx(g["rf_est"][0], rel=1e-12)
    bf = O.fast_range_finder(A[:, :16], 5, 4)
    assert np.abs(bf.Q - g["rf_fast_Q"]).max() <= 1e-12
    assert bf.diagnostics["max_imag_sample"] == pytest.approx(g["rf_fast_maximag"][0], rel=1e-12)


def test_cfg1_oracle_matches_reference(golden):
    g = golden("cfg1")
    c = workloads.CONFIGS[1]
    A, _ = workloads.build_cfg1()
    assert np.array_equal(A[:4, :8], g["A_head"])
    op = O.Dense(A)
    basis, f, est = O.rsvd(op, c.k, c.p, c.q, c.seed)
    assert np.abs(f.sigma - g["sigma"]).max() / g["sigma"][0] <= 1e-13
    assert np.all(np.abs(f.sigma - g["sigma"]) <= 1e-10 * g["sigma"])
    assert est == pytest.approx(g["est"][0], rel=1e-10)
    assert basis.passes == g["passes"][0] and basis.Q.shape[1] == g["rank"][0]
    assert np.abs(basis.Q[:8] - g["Q_head"]).max() <= 1e-12
    assert np.abs(f.U[:8] - g["U_head"]).max() <= 1e-11
    assert np.abs(f.V[:8] - g["V_head"]).max() <= 1e-11
    assert [op.counters.matvecs, op.counters.adjoint_matvecs, op.counters.passes,
            op.counters.flops] == list(g["counters"])


def test_cfg5_reduced_oracle_matches_reference(golden):
    g = golden("cfg5s")
    c = workloads.CONFIGS[5]
    S, L, R = workloads.build_cfg5(n=1 << 16)
    assert S.nnz == g["nnz"][0]
    op = O.SparsePlusLowRank(S, L, R)
    basis, f, est = O.rsvd(op, c.k, c.p, c.q, c.seed)
    top = g["sigma"] > 1e-6 * g["sigma"][0]
    assert np.all(np.abs(f.sigma - g["sigma"])[top] <= 1e-10 * g["sigma"][top])
    assert est == pytest.approx(g["est"][0], rel=1e-6)
    assert basis.passes == g["passes"][0]


def test_gsrft_oracle_matches_reference(golden):
    """Givens-chain SRFT (reference sketch.py:221-337): draws bitwise, the
    apply (power-of-two and not) and the gsrft range finder."""
    g = golden("kats")
    d = O.gsrft_operator(16, 4, 2)
    for f in ("d_outer", "perm_outer", "thetas_outer", "d_mid", "perm_inner", "thetas_inner",
              "d_inner", "picks"):
        assert np.array_equal(getattr(d, f), g[f"gsrft16_{f}"]), f
    assert np.abs(O.gsrft_apply(g["gsrft_A"], d) - g["gsrft_Y"]).max() <= 1e-13
    Y = O.gsrft_apply(g["gsrft12_A"], O.gsrft_operator(12, 5, 7))
    assert np.abs(Y - g["gsrft12_Y"]).max() <= 1e-13
    b = O.fast_range_finder(g["rf_A"][:, :16], 5, 4, kind="gsrft")
    assert np.abs(b.Q - g["rf_gsrft_Q"]).max() <= 1e-12


def test_adaptive_oracle_matches_reference(golden):
    """Alg 4.2 fixed-precision finder (reference rangefinder.py:89-166)."""
    g = golden("kats")
    for blk in (1, 4):
        b = O.adaptive_range_finder(g["ad_A"], 1e-3, r=10, seed=5, block=blk)
        meta = g[f"ad{blk}_meta"]
        assert b.Q.shape == g[f"ad{blk}_Q"].shape
        assert np.abs(b.Q - g[f"ad{blk}_Q"]).max() <= 1e-12
        assert [b.samples_used, b.passes, float(b.saturated), b.probe_matvecs] == \
            [meta[0], meta[1], meta[3], meta[4]]
        assert b.est_error == pytest.approx(meta[2], rel=1e-10)
    b = O.adaptive_range_finder(g["ad_A"][:, :8], 1e-12, r=4, seed=2)
    assert b.saturated and b.Q.shape == g["ad_sat_Q"].shape
    assert np.abs(b.Q - g["ad_sat_Q"]).max() <= 1e-12


def test_stageb_hermitian_routes(golden):
    """direct_eig_hermitian / small_eig_hermitian / eig_nystrom restatements
    against the reference (factor.py:168-191,300-335, core.py:233-294)."""
    g = golden("stageb")
    f = O.direct_eig_hermitian(g["eig_A"], g["eig_Q"])
    assert np.abs(f.lam - g["eig_lam"]).max() <= 1e-13 * np.abs(g["eig_lam"]).max()
    assert np.abs(f.compose() - g["eig_comp"]).max() <= 1e-13
    assert np.allclose(O.direct_eig_hermitian(np.diag([3.0, -2.0, 1.0]), np.eye(3)).lam,
                       g["eig_diag_lam"], rtol=0, atol=1e-15)
    f = O.direct_eig_hermitian(g["eigc_A"], g["eigc_Q"])
    assert np.abs(f.lam - g["eigc_lam"]).max() <= 1e-13 * np.abs(g["eigc_lam"]).max()
    assert np.abs(f.compose() - g["eigc_comp"]).max() <= 1e-13
    _, lam = O.small_eig_hermitian(g["seig_B"])
    assert np.abs(lam - g["seig_lam"]).max() <= 1e-13
    for tag in ("nys_rank", "nys_exp", "nys_pow"):
        f, F = O.eig_nystrom(g[f"{tag}_H"], g[f"{tag}_Q"])
        scale = np.abs(g[f"{tag}_lam"]).max()
        assert np.abs(f.lam - g[f"{tag}_lam"]).max() <= 1e-12 * scale
        assert np.abs(f.compose() - g[f"{tag}_comp"]).max() <= 1e-12 * scale
        assert np.abs(F @ F.conj().T - g[f"{tag}_FF"]).max() <= 1e-12 * scale
    f, _ = O.eig_nystrom(np.diag([1.0, 0.5, -0.8]), np.eye(3))
    assert f.diagnostics.get("not_psd_fallback") and g["nys_fb_flag"][0] == 1.0
    assert np.allclose(f.lam, g["nys_fb_lam"], rtol=0, atol=1e-15)
    with pytest.raises(ValueError):
        O.direct_eig_hermitian(np.random.default_rng(13).standard_normal((10, 10)),
                               np.eye(10)[:, :3])


def test_oracle_one_pass_and_streaming(golden, tmp_path):
    """The oracle's one-pass factorizations and row-block streaming against
    the reference's own outputs (tests/golden/onepass.npz)."""
    g = golden("onepass")
    b = O.sample_bundle_two_sided(g["gen_A"], 15, seed=6)
    f = O.svd_one_pass_general(b)
    assert np.abs(f.sigma - g["gen_sigma"]).max() <= 1e-10 * g["gen_sigma"][0]
    assert np.abs(f.U * f.sigma @ f.V.conj().T - g["gen_comp"]).max() <= 1e-9
    b = O.sample_bundle_two_sided(g["gen2_A"], 20, ell_tilde=24, seed=9)
    f = O.svd_one_pass_general(b)
    assert np.abs(f.sigma - g["gen2_sigma"]).max() <= 1e-10 * g["gen2_sigma"][0]
    b = O.sample_bundle_two_sided(g["gen2_A"], 20, ell_tilde=24, seed=9, rank=10)
    f = O.svd_one_pass_general(b)
    assert np.abs(f.sigma - g["gen2r_sigma"]).max() <= 1e-10 * g["gen2r_sigma"][0]
    for tag, rank in (("herm", None), ("herm2", 10)):
        H = g[f"{tag}_H"]
        b = O.sample_bundle(H, 16 if tag == "herm" else 20, seed=5, rank=rank)
        e = O.eig_one_pass(b)
        assert np.abs(e.lam - g[f"{tag}_lam"]).max() <= 1e-9 * np.abs(g[f"{tag}_lam"]).max()
        assert e.diagnostics["tau_min"] == pytest.approx(g[f"{tag}_tau"][0], rel=1e-9)
    for tag, br, ell in (("st", 8, 6), ("stc", 5, 4)):
        p = tmp_path / f"{tag}.bin"
        O.write_matrix_binary(g[f"{tag}_A"], p)
        assert np.array_equal(np.frombuffer(p.read_bytes()[:64], dtype=np.uint8), g[f"{tag}_bytes"])
        sb = O.streamed_sample_bundle(str(p), br, ell, seed=4)
        assert np.array_equal(sb.Omega, g[f"{tag}_Om"])
        assert np.array_equal(sb.Y, g[f"{tag}_Y"]) and np.array_equal(sb.Y_tilde, g[f"{tag}_Yt"])
        assert np.abs(sb.Q - g[f"{tag}_Q"]).max() <= 1e-13


def test_oracle_row_id_and_extraction(golden):
    """The oracle's interpolative decomposition / row extraction against the
    reference's outputs (tests/golden/rowid.npz)."""
    g = golden("rowid")
    ks = {"small": 2, "dup": 2, "lowrank": 5}
    names = sorted({k[4:-2] for k in g if k.startswith("rid_") and k.endswith("_M")})
    for name in names:
        M = g[f"rid_{name}_M"]
        J, X = O.row_id(M, ks.get(name, M.shape[1]))
        assert np.array_equal(J, g[f"rid_{name}_J"]), name
        assert np.abs(X - g[f"rid_{name}_X"]).max() <= 1e-10, name
    f = O.svd_via_row_extraction(g["sre2_A"], g["sre2_Q"])
    assert np.abs(f.sigma - g["sre2_sigma"]).max() <= 1e-10 * g["sre2_sigma"][0]
