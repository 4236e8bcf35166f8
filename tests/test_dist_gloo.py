"""Row-sharded multi-rank path on CPU: world_size 2 over
gloo, the host logic of paper_0909_4061_b200.dist driven through the
test backend (tests/dist_np_backend.py), checked against the single-process
oracle rsvd on the whole matrix.  The GPU backend runs the same functions
with NCCL; only the primitives differ."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lowrank_oracle as orc

import workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _matrix(case):
    rng = np.random.default_rng(7)
    if case == "decay":
        m, n = 300, 160
        s = np.exp(-np.arange(n) / 8.0)
        return workloads.synthetic_explicit(m, n, s, 3)[0]
    if case == "rank5":           # exact rank 5 < ell: drops -> CGS2 fallback
        return rng.standard_normal((260, 5)) @ rng.standard_normal((5, 90))
    if case == "complex":
        m, n = 220, 120
        U, _ = np.linalg.qr(rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)))
        V, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        s = np.exp(-np.arange(n) / 6.0)
        return (U * s) @ V.conj().T
    if case == "zero":
        return np.zeros((64, 40))
    raise ValueError(case)


CASES = {  # name -> (k, p, q, row split for rank 0)
    "decay": (10, 6, 2, 170),
    "rank5": (8, 4, 1, 101),
    "complex": (12, 6, 1, 111),
    "zero": (4, 2, 1, 30),
}


def _worker(rank, world, port, case, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_0909_4061_b200.dist import Comm, dist_randomized_svd
        from dist_np_backend import TorchCpuBackend
        A = _matrix(case)
        k, p, q, cut = CASES[case]
        rows = [(0, cut), (cut, A.shape[0])][rank]
        A_local = torch.from_numpy(np.ascontiguousarray(A[rows[0]:rows[1]]))
        res = dist_randomized_svd(A_local, A.shape[1], k, p, q, seed=5, comm=Comm(),
                                  be=TorchCpuBackend())
        torch.save({"Q": res.Q, "U": res.U, "sigma": res.sigma, "V": res.V, "est": res.est,
                    "rows": rows}, os.path.join(outdir, f"r{rank}.pt"))
    finally:
        dist.destroy_process_group()


def _run(case):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), case, d), nprocs=2, join=True)
        return [torch.load(os.path.join(d, f"r{r}.pt")) for r in range(2)]


@pytest.mark.parametrize("case", list(CASES))
def test_row_sharded_rsvd_matches_oracle(case):
    A = _matrix(case)
    k, p, q, _ = CASES[case]
    basis, f, est = orc.rsvd(A, k, p, q, seed=5)
    outs = _run(case)
    # replicated outputs identical on both ranks
    for key in ("sigma", "V"):
        assert torch.equal(outs[0][key], outs[1][key]), key
    assert outs[0]["est"] == outs[1]["est"]
    Q = np.vstack([o["Q"].numpy() for o in outs])
    U = np.vstack([o["U"].numpy() for o in outs])
    S = outs[0]["sigma"].numpy()
    V = outs[0]["V"].numpy()
    assert Q.shape[1] == basis.Q.shape[1]                      # same rank decision
    if Q.shape[1] == 0:
        assert est == 0.0 or est is None or outs[0]["est"] == 0.0
        return
    assert np.allclose(Q.conj().T @ Q, np.eye(Q.shape[1]), atol=1e-12)
    # same subspace as the oracle basis (principal angles ~ 0)
    assert np.linalg.norm(Q - basis.Q @ (basis.Q.conj().T @ Q)) < 1e-9
    # sigma: relative 1e-10 (fp64 tolerance of north_star)
    s_ref = f.sigma
    assert np.max(np.abs(S - s_ref) / s_ref[0]) < 1e-10
    # U, V columns with sigma gaps: same vectors (sign convention identical)
    gap = np.abs(np.diff(s_ref)) > 1e-6 * s_ref[0]
    for j in range(min(len(S) - 1, 6)):
        if gap[j] and (j == 0 or gap[j - 1]):
            assert np.linalg.norm(U[:, j] - f.U[:, j]) < 1e-7
            assert np.linalg.norm(V[:, j] - f.V[:, j]) < 1e-7
    # estimate: relative 1e-8, or roundoff level of ||A|| when the tail is exact zero
    assert abs(outs[0]["est"] - est) <= 1e-8 * est + 1e-12 * s_ref[0]
    # reconstruction from the sharded factors
    A_hat = (U * S) @ V.conj().T
    assert np.linalg.norm(A - A_hat, 2) <= 10 * max(est, 1e-12)


def _sparse_case():
    import scipy.sparse as sp
    n, per_row, r = 3000, 12, 4
    g = np.random.default_rng(41)
    cols = g.integers(0, n, size=(n, per_row))
    vals = g.standard_normal((n, per_row))
    rows = np.repeat(np.arange(n), per_row)
    S = sp.csr_matrix((vals.ravel(), (rows, cols.ravel())), shape=(n, n))
    S.sum_duplicates()
    S.sort_indices()
    L = 10.0 * g.standard_normal((n, r))
    R = 10.0 * g.standard_normal((n, r))
    return S, L, R


def _sparse_worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_0909_4061_b200.dist import Comm, dist_randomized_svd_operator, row_range
        from dist_np_backend import TorchCpuBackend
        S, L, R = _sparse_case()
        n = S.shape[0]
        a, b = row_range(n, rank, world)
        op_local = (S[a:b], L[a:b], R)
        res = dist_randomized_svd_operator(op_local, n, 6, 4, 2, seed=5, comm=Comm(),
                                           be=TorchCpuBackend())
        torch.save({"Q": res.Q, "U": res.U, "sigma": res.sigma, "V": res.V, "est": res.est,
                    "passes": res.passes}, os.path.join(outdir, f"s{rank}.pt"))
    finally:
        dist.destroy_process_group()


def test_row_sharded_sparse_rsvd_matches_oracle():
    """Config 5's sharded path (dist_randomized_svd_operator): S + L R^T split
    by rows over 2 gloo ranks, n-side panels sharded too (all-gather before
    A_r X, reduce-scatter after A_r^H Y), against the oracle's rsvd of the
    whole operator."""
    S, L, R = _sparse_case()
    basis, f, est = orc.rsvd(orc.SparsePlusLowRank(S, L, R), 6, 4, 2, seed=5)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_sparse_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        outs = [torch.load(os.path.join(d, f"s{r}.pt")) for r in range(2)]
    assert torch.equal(outs[0]["sigma"], outs[1]["sigma"])
    assert outs[0]["passes"] == basis.passes == 6
    S_ = outs[0]["sigma"].numpy()
    assert np.max(np.abs(S_ - f.sigma) / f.sigma[0]) < 1e-10
    Q = np.vstack([o["Q"].numpy() for o in outs])
    U = np.vstack([o["U"].numpy() for o in outs])
    V = np.vstack([o["V"].numpy() for o in outs])
    assert np.linalg.norm(Q - basis.Q @ (basis.Q.T @ Q)) < 1e-9
    for j in range(4):
        assert np.linalg.norm(U[:, j] - f.U[:, j]) < 1e-7
        assert np.linalg.norm(V[:, j] - f.V[:, j]) < 1e-7
    assert abs(outs[0]["est"] - est) <= 1e-8 * est
