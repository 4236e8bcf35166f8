"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (the reference lives at /root/reference and
does not travel to the GPU box):

    python tests/golden/make_golden.py [name ...]

Writes small .npz fixtures next to this script.  Each fixture stores the
inputs' seeds/recipes (matrices are regenerated from seeds by workloads.py)
and the reference's outputs: singular values, estimator values, pass counts
and leading slices of Q/U/V.  tests/test_oracle_golden.py pins the oracle
to these; tests/test_gpu_parity.py pins the CUDA path to them.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import lowrank  # noqa: E402  (the reference)
from lowrank import core, factor, rangefinder, sketch  # noqa: E402
from lowrank.oracle import SyntheticSpec, synthetic_matrix  # noqa: E402

import workloads  # noqa: E402


def save(name, **arrs):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrs)
    print(f"wrote {path} ({os.path.getsize(path)} B)", flush=True)


def g_kats():
    out = {}
    # Philox draws (sketch.py:32-42,96-100; rangefinder.py:78)
    out["gauss_7x3_s11"] = sketch.gaussian_matrix(7, 3, 11)
    out["probe_6x2_s5"] = sketch.rng_for(5, 0x70726F62).standard_normal((6, 2))
    op = sketch.srft_operator(64, 8, 3)
    out["srft64_d"], out["srft64_picks"] = op.d, op.picks
    op = sketch.srft_operator(8192, 120, 3)
    out["srft8192_d_head"], out["srft8192_picks"] = op.d[:64], op.picks
    out["srft8192_d_sum"] = np.array([op.d.sum()])
    # orthonormalize_double_gs (core.py:84-115) KATs, test_core.py:75-93
    out["dgs_collinear"] = core.orthonormalize_double_gs(np.array([[1.0, 2.0], [0.0, 0.0]]))
    rng = np.random.default_rng(11)
    Y = rng.standard_normal((100, 10))
    Y[:, 1] = 1e-14 * Y[:, 0]
    out["dgs_neardep_Y"], out["dgs_neardep_Q"] = Y, core.orthonormalize_double_gs(Y)
    rng = np.random.default_rng(12)
    Y = rng.standard_normal((40, 12))
    out["dgs_rand_Y"], out["dgs_rand_Q"] = Y, core.orthonormalize_double_gs(Y)
    Yc = rng.standard_normal((30, 7)) + 1j * rng.standard_normal((30, 7))
    out["dgs_cplx_Y"], out["dgs_cplx_Q"] = Yc, core.orthonormalize_double_gs(Yc)
    # small_svd (core.py:199-230) KATs, test_core.py:144-184
    f = core.small_svd(np.array([[1.0, 1.0], [0.0, 1.0]]))
    out["svd_golden_s"] = f.sigma
    rng = np.random.default_rng(8)
    B = rng.standard_normal((7, 9))
    f = core.small_svd(B)
    out["svd_rand_B"], out["svd_rand_U"], out["svd_rand_s"], out["svd_rand_V"] = B, f.U, f.sigma, f.V
    Bc = rng.standard_normal((6, 11)) + 1j * rng.standard_normal((6, 11))
    f = core.small_svd(Bc)
    out["svd_cplx_B"], out["svd_cplx_U"], out["svd_cplx_s"], out["svd_cplx_V"] = Bc, f.U, f.sigma, f.V
    # direct_svd KAT (tests/test_factor.py:46-51)
    f = factor.direct_svd(core.DenseOperator(np.diag([5.0, 4.0, 3.0, 2.0, 1.0])), np.eye(5)[:, :3])
    out["dsvd_diag_s"] = f.sigma
    # dft (sketch.py:179-200), test_sketch.py:90-107
    out["dft_n2"] = sketch.dft(np.array([1.0, 0.0]))
    out["dft_n4"] = sketch.dft(np.ones(4))
    rng = np.random.default_rng(16)
    v = rng.standard_normal((3, 16)) + 1j * rng.standard_normal((3, 16))
    out["dft16_in"], out["dft16_out"] = v, sketch.dft(v, axis=1)
    v = rng.standard_normal((2, 12))
    out["dft12_in"], out["dft12_out"] = v, sketch.dft(v, axis=1)
    # srft_apply (sketch.py:306-320), test_sketch.py:147-151
    rng = np.random.default_rng(6)
    A = rng.standard_normal((16, 16))
    op = sketch.srft_operator(16, 4, 1)
    out["srft_A"], out["srft_Y"] = A, sketch.srft_apply(A, op)
    # small range-finder runs (rangefinder.py), exercised at every entry point
    rng = np.random.default_rng(10)
    A = rng.standard_normal((25, 18))
    out["rf_A"] = A
    b = rangefinder.randomized_range_finder(A, 6, 11)
    out["rf_basic_Q"] = b.Q
    b = rangefinder.power_iteration_range(A, 6, 2, 11)
    out["rf_power_Q"] = b.Q
    b = rangefinder.subspace_iteration_range(A, 6, 2, 11)
    out["rf_subspace_Q"] = b.Q
    f = factor.direct_svd(A, b.Q)
    out["rf_dsvd_U"], out["rf_dsvd_s"], out["rf_dsvd_V"] = f.U, f.sigma, f.V
    out["rf_est"] = np.array([rangefinder.posterior_error_estimate(A, b.Q, seed=3)])
    b = rangefinder.fast_range_finder(A[:, :16], 5, 4)
    out["rf_fast_Q"] = b.Q
    out["rf_fast_maximag"] = np.array([b.diagnostics["max_imag_sample"]])
    # Givens-chain SRFT (sketch.py:221-337): draws, apply (power-of-two and
    # not), and the fast range finder with kind="gsrft"
    g = sketch.gsrft_operator(16, 4, 2)
    for f in ("d_outer", "perm_outer", "thetas_outer", "d_mid", "perm_inner", "thetas_inner",
              "d_inner", "picks"):
        out[f"gsrft16_{f}"] = getattr(g, f)
    rng = np.random.default_rng(12)
    A = rng.standard_normal((5, 16)) + 1j * rng.standard_normal((5, 16))
    out["gsrft_A"], out["gsrft_Y"] = A, sketch.gsrft_apply(A, g)
    A = rng.standard_normal((4, 12))
    out["gsrft12_A"], out["gsrft12_Y"] = A, sketch.gsrft_apply(A, sketch.gsrft_operator(12, 5, 7))
    b = rangefinder.fast_range_finder(out["rf_A"][:, :16], 5, 4, kind="gsrft")
    out["rf_gsrft_Q"] = b.Q
    # adaptive fixed-precision range finder (rangefinder.py:89-166), single and
    # blocked draws, on a matrix with a decaying spectrum
    rng = np.random.default_rng(13)
    U = np.linalg.qr(rng.standard_normal((60, 40)))[0]
    V = np.linalg.qr(rng.standard_normal((50, 40)))[0]
    A = (U * np.exp(-np.arange(40) / 3.0)) @ V.T
    out["ad_A"] = A
    for blk in (1, 4):
        b = rangefinder.adaptive_range_finder(A, 1e-3, r=10, seed=5, block=blk)
        out[f"ad{blk}_Q"] = b.Q
        out[f"ad{blk}_meta"] = np.array([b.samples_used, b.passes, b.est_error,
                                         float(b.saturated), b.probe_matvecs])
    b = rangefinder.adaptive_range_finder(A[:, :8], 1e-12, r=4, seed=2)
    out["ad_sat_Q"] = b.Q
    out["ad_sat_meta"] = np.array([b.samples_used, b.passes, b.est_error, float(b.saturated),
                                   b.probe_matvecs])
    save("kats", **out)


def run_cfg(A_or_op, k, p, q, seed, sketch_kind="gauss", A_dense=None):
    op = core.as_operator(A_or_op)
    ell = k + p
    t0 = time.perf_counter()
    if sketch_kind == "gauss":
        basis = (rangefinder.subspace_iteration_range(op, ell, q, seed) if q > 0
                 else rangefinder.randomized_range_finder(op, ell, seed))
    else:
        basis = rangefinder.fast_range_finder(A_dense, ell, seed, kind="srft")
    f = factor.direct_svd(op, basis.Q)
    t1 = time.perf_counter()
    est = rangefinder.posterior_error_estimate(op, basis.Q, r=10, alpha=10.0, seed=seed + 13)
    t2 = time.perf_counter()
    print(f"  reference stage A + direct_svd {t1 - t0:.2f}s, estimator {t2 - t1:.2f}s", flush=True)
    return dict(sigma=f.sigma, est=np.array([est]), passes=np.array([basis.passes]),
                samples=np.array([basis.samples_used]), rank=np.array([basis.Q.shape[1]]),
                Q_head=basis.Q[:8], U_head=f.U[:8], V_head=f.V[:8],
                Q_colsum=basis.Q.sum(axis=0), U_colsum=f.U.sum(axis=0), V_colsum=f.V.sum(axis=0),
                counters=np.array([op.counters.matvecs, op.counters.adjoint_matvecs,
                                   op.counters.passes, op.counters.flops], dtype=np.int64),
                t_ref=np.array([t1 - t0, t2 - t1]))


def g_cfg1():
    c = workloads.CONFIGS[1]
    A, s = synthetic_matrix(SyntheticSpec(c.m, c.n, "explicit", workloads.spectrum(1, c.n), c.seed))
    Aw, _ = workloads.build_cfg1()
    assert np.array_equal(A, Aw), "workloads.build_cfg1 must reproduce the reference builder"
    save("cfg1", **run_cfg(A, c.k, c.p, c.q, c.seed), A_head=A[:4, :8], A_fro=np.array([np.linalg.norm(A)]))


def g_cfg2():
    c = workloads.CONFIGS[2]
    t0 = time.time()
    A, _ = synthetic_matrix(SyntheticSpec(c.m, c.n, "explicit", workloads.spectrum(2, c.n), c.seed))
    print(f"  cfg2 A built in {time.time() - t0:.0f}s", flush=True)
    save("cfg2", **run_cfg(A, c.k, c.p, c.q, c.seed), A_head=A[:4, :8], A_fro=np.array([np.linalg.norm(A)]))


def g_cfg3():
    c = workloads.CONFIGS[3]
    A = workloads.build_cfg3()
    save("cfg3", **run_cfg(A, c.k, c.p, c.q, c.seed, "srft", A_dense=A), A_head=A[:4, :8],
         A_fro=np.array([np.linalg.norm(A.astype(np.complex128))]))


def g_cfg4s():
    """cfg4 recipe at one 65536-row block (the full 2^20 rows need a 32 GiB
    fp64 upcast and ~15 min of CGS2 in the reference)."""
    c = workloads.CONFIGS[4]
    A, _ = workloads.build_cfg4_host(m=65536)
    save("cfg4s", **run_cfg(A, c.k, c.p, c.q, c.seed), A_head=A[:4, :8],
         A_fro=np.array([np.linalg.norm(A.astype(np.float64))]))


class _CsrPlusLowRank(core.MatVecOperator):
    """A user MatVecOperator plug-in over scipy CSR (the
    reference has no sparse code; this is the oracle the survey prescribes)."""

    def __init__(self, S, L, R):
        super().__init__(*S.shape)
        self.S, self.St, self.L, self.R = S, S.T.tocsr(), L, R

    def _apply(self, X):
        return self.S @ X + self.L @ (self.R.T @ X)

    def _apply_adjoint(self, Y):
        return self.St @ Y + self.R @ (self.L.T @ Y)


def g_cfg5s():
    """cfg5 recipe at n = 2^16 rows/cols."""
    c = workloads.CONFIGS[5]
    S, L, R = workloads.build_cfg5(n=1 << 16)
    op = _CsrPlusLowRank(S, L, R)
    save("cfg5s", **run_cfg(op, c.k, c.p, c.q, c.seed), nnz=np.array([S.nnz]))


def g_stageb():
    """Hermitian Stage-B routes (factor.py:168-191,300-335) on small inputs;
    the matrices are stored (they are tiny)."""
    from lowrank.oracle import synthetic_psd
    out = {}
    rng = np.random.default_rng(12)
    G = rng.standard_normal((18, 18))
    A = 0.5 * (G + G.T)
    b = rangefinder.randomized_range_finder(core.DenseOperator(A), 6, seed=0)
    f = factor.direct_eig_hermitian(core.DenseOperator(A), b.Q)
    out.update(eig_A=A, eig_Q=b.Q, eig_lam=f.lam, eig_comp=f.compose())
    f = factor.direct_eig_hermitian(core.DenseOperator(np.diag([3.0, -2.0, 1.0])), np.eye(3))
    out["eig_diag_lam"] = f.lam
    Gc = rng.standard_normal((16, 16)) + 1j * rng.standard_normal((16, 16))
    Ac = 0.5 * (Gc + Gc.conj().T)
    b = rangefinder.randomized_range_finder(core.DenseOperator(Ac), 5, seed=1)
    f = factor.direct_eig_hermitian(core.DenseOperator(Ac), b.Q)
    out.update(eigc_A=Ac, eigc_Q=b.Q, eigc_lam=f.lam, eigc_comp=f.compose())
    out["seig_B"] = rng.standard_normal((9, 9))
    V, lam = core.small_eig_hermitian(out["seig_B"])
    out["seig_lam"] = lam
    for tag, (kind, par, sd, ell, qs) in {"nys_rank": ("exact_rank", 4, 17, 6, 1),
                                         "nys_exp": ("exp_decay", 0.7, 18, 6, 4),
                                         "nys_pow": ("power_decay", 1.5, 3, 7, 3)}.items():
        H, _ = synthetic_psd(25 if tag != "nys_pow" else 24, kind, par, seed=sd)
        b = rangefinder.randomized_range_finder(core.DenseOperator(H), ell, seed=qs)
        f, fac = factor.eig_nystrom(core.DenseOperator(H), b.Q)
        out.update({f"{tag}_H": H, f"{tag}_Q": b.Q, f"{tag}_lam": f.lam,
                    f"{tag}_comp": f.compose(), f"{tag}_FF": fac.F @ fac.F.conj().T})
    f, fac = factor.eig_nystrom(core.DenseOperator(np.diag([1.0, 0.5, -0.8])), np.eye(3))
    out["nys_fb_lam"] = f.lam
    out["nys_fb_flag"] = np.array([float(bool(f.diagnostics.get("not_psd_fallback")))])
    save("stageb", **out)


def g_onepass():
    """One-pass sketches (reference factor.py:123-147,338-401) and the
    LRKMAT00 / row-block streaming path (io.py:178-204,319-430)."""
    import tempfile
    from lowrank import io as rio
    from lowrank.oracle import synthetic_psd
    out = {}
    A, _ = synthetic_matrix(SyntheticSpec(m=40, n=30, kind="exact_rank", param=5, seed=20))
    b = factor.sample_bundle_two_sided(A, 15, seed=6)
    f = factor.svd_one_pass_general(b)
    out.update(gen_A=A, gen_Q=b.Q, gen_Qt=b.Q_tilde, gen_Y=b.Y, gen_Yt=b.Y_tilde,
               gen_sigma=f.sigma, gen_comp=f.compose())
    rng = np.random.default_rng(23)
    A2 = (rng.standard_normal((120, 12)) * np.exp(-np.arange(12) / 3.0)) @ rng.standard_normal((12, 90))
    A2 += 1e-3 * rng.standard_normal((120, 90))
    b = factor.sample_bundle_two_sided(A2, 20, ell_tilde=24, seed=9)
    f = factor.svd_one_pass_general(b)
    out.update(gen2_A=A2, gen2_sigma=f.sigma, gen2_comp=f.compose(), gen2_Q=b.Q, gen2_Qt=b.Q_tilde)
    b = factor.sample_bundle_two_sided(A2, 20, ell_tilde=24, seed=9, rank=10)
    f = factor.svd_one_pass_general(b)
    out.update(gen2r_sigma=f.sigma, gen2r_comp=f.compose())
    H, _ = synthetic_psd(40, "exact_rank", 6, seed=19)
    b = factor.sample_bundle(core.DenseOperator(H), 16, seed=5)
    f = factor.eig_one_pass(b)
    out.update(herm_H=H, herm_Q=b.Q, herm_lam=f.lam, herm_comp=f.compose(),
               herm_tau=np.array([f.diagnostics["tau_min"]]))
    H2, _ = synthetic_psd(40, "exp_decay", 0.9, seed=4)
    b = factor.sample_bundle(core.DenseOperator(H2), 20, seed=5, rank=10)
    f = factor.eig_one_pass(b)
    out.update(herm2_H=H2, herm2_lam=f.lam, herm2_tau=np.array([f.diagnostics["tau_min"]]),
               herm2_comp=f.compose())
    # streamed bundle of a stored matrix (block_rows 8), complex too
    rng = np.random.default_rng(10)
    S = rng.standard_normal((64, 32))
    Sc = rng.standard_normal((33, 20)) + 1j * rng.standard_normal((33, 20))
    with tempfile.TemporaryDirectory() as d:
        for tag, M, br, ell in (("st", S, 8, 6), ("stc", Sc, 5, 4)):
            pth = os.path.join(d, f"{tag}.bin")
            rio.write_matrix_binary(M, pth)
            sb = rio.streamed_sample_bundle(rio.stream_row_blocks(pth, br), ell=ell, seed=4)
            out.update({f"{tag}_A": M, f"{tag}_Y": sb.Y, f"{tag}_Yt": sb.Y_tilde, f"{tag}_Q": sb.Q,
                        f"{tag}_Qt": sb.Q_tilde, f"{tag}_Om": sb.Omega, f"{tag}_Omt": sb.Omega_tilde,
                        f"{tag}_bytes": np.frombuffer(open(pth, "rb").read()[:64], dtype=np.uint8)})
    save("onepass", **out)


def g_rowid():
    """Interpolative decomposition and row extraction (reference
    factor.py:198-296, pivoted QR core.py:133-186)."""
    from lowrank.oracle import synthetic_psd
    out = {}
    cases = {"small": np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0]]),
             "dup": np.array([[1.0, 2.0], [1.0, 2.0], [0.0, 1.0]])}
    rng = np.random.default_rng(4)
    for t in range(12):
        cases[f"rand{t}"] = rng.standard_normal((25, 6))
    rng = np.random.default_rng(5)
    cases["lowrank"] = rng.standard_normal((15, 3)) @ rng.standard_normal((3, 8))
    rng = np.random.default_rng(7)
    cases["cplx"] = rng.standard_normal((14, 4)) + 1j * rng.standard_normal((14, 4))
    rng = np.random.default_rng(3)
    cases["tall"] = np.linalg.qr(rng.standard_normal((3000, 40)))[0]
    ks = {"small": 2, "dup": 2, "lowrank": 5}
    for name, M in cases.items():
        k = ks.get(name, M.shape[1])
        f = factor.row_id(M, k)
        if name == "tall":      # regenerated by the tests (same rng, numpy QR)
            out["rid_tall_J"], out["rid_tall_Xhead"] = f.J, f.X[:64]
            continue
        out[f"rid_{name}_M"], out[f"rid_{name}_J"], out[f"rid_{name}_X"] = M, f.J, f.X
    rng = np.random.default_rng(6)
    M = rng.standard_normal((12, 4)) @ rng.standard_normal((4, 18))
    c = factor.column_id(M, 4)
    out.update(cid_M=M, cid_J=c.J, cid_X=c.X)
    A, _ = synthetic_matrix(SyntheticSpec(m=30, n=25, kind="exact_rank", param=5, seed=8))
    b = rangefinder.randomized_range_finder(core.DenseOperator(A), 5, seed=1)
    f = factor.svd_via_row_extraction(A, b.Q)
    out.update(sre_A=A, sre_Q=b.Q, sre_sigma=f.sigma, sre_comp=f.compose())
    rng = np.random.default_rng(9)
    A = rng.standard_normal((50, 50))
    b = rangefinder.randomized_range_finder(core.DenseOperator(A), 8, seed=3)
    f = factor.svd_via_row_extraction(A, b.Q)
    out.update(sre2_A=A, sre2_Q=b.Q, sre2_sigma=f.sigma, sre2_comp=f.compose())
    rng = np.random.default_rng(11)
    A = rng.standard_normal((30, 30))
    Y = A @ rng.standard_normal((30, 6))
    f = factor.svd_via_row_extraction(A, Y)
    out.update(sre3_A=A, sre3_Y=Y, sre3_sigma=f.sigma, sre3_comp=f.compose())
    H, _ = synthetic_psd(30, "exact_rank", 5, seed=14)
    b = rangefinder.randomized_range_finder(core.DenseOperator(H), 5, seed=2)
    f = factor.eig_via_row_extraction(H, b.Q)
    out.update(ere_H=H, ere_Q=b.Q, ere_lam=f.lam, ere_comp=f.compose())
    save("rowid", **out)


ALL = {"rowid": g_rowid, "onepass": g_onepass, "kats": g_kats, "stageb": g_stageb, "cfg1": g_cfg1, "cfg3": g_cfg3, "cfg4s": g_cfg4s, "cfg5s": g_cfg5s,
       "cfg2": g_cfg2}

if __name__ == "__main__":
    names = sys.argv[1:] or list(ALL)
    for nm in names:
        print(f"[{nm}]", flush=True)
        ALL[nm]()
