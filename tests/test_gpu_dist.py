"""Row-sharded path on the GPU backend.

Only one GPU is available to the tests, so the multi-rank cases run two
ranks as two host threads on one device, each on its own CUDA stream, with a
host-side all-reduce (ThreadComm: D2H, barrier, fixed-order sum, H2D) -- no
kernel ever waits on another rank's kernel.  The NCCL communicator itself is
exercised at world_size 1 through the public entry (sharded_randomized_svd).
"""

import socket
import threading

import numpy as np
import pytest

from oracle import lowrank_oracle as orc

pytestmark = pytest.mark.gpu


class ThreadComm:
    def __init__(self, world, rank, shared):
        self.world, self.rank, self.shared = world, rank, shared

    def _reduce(self, t, fn):
        import torch
        sh = self.shared
        sh["buf"][self.rank] = t.cpu().numpy().copy()
        sh["bar"].wait()
        out = sh["buf"][0].copy()
        for r in range(1, self.world):
            out = fn(out, sh["buf"][r])
        sh["bar"].wait()
        t.copy_(torch.from_numpy(out))
        return t

    def allreduce(self, t):
        return self._reduce(t, lambda a, b: a + b)

    def allreduce_max(self, t):
        return self._reduce(t, np.maximum)


def _run_threads(A, cuts, k, p, q, seed, dtype=None, sketch="gauss"):
    import torch
    from paper_0909_4061_b200 import DenseOperator
    from paper_0909_4061_b200.dist import GpuBackend, dist_randomized_svd
    world = len(cuts) - 1
    shared = {"buf": [None] * world, "bar": threading.Barrier(world)}
    out = [None] * world
    errs = []

    def work(r):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                blk = np.ascontiguousarray(A[cuts[r]:cuts[r + 1]])
                op = DenseOperator(torch.from_numpy(blk).cuda() if dtype is None
                                   else torch.from_numpy(blk).cuda().to(dtype))
                comm = ThreadComm(world, r, shared)
                amax = None
                if op.array.dtype in (torch.float32, torch.complex64):
                    t = torch.tensor([op.amax], dtype=torch.float64, device="cuda")
                    amax = float(comm.allreduce_max(t).item())
                res = dist_randomized_svd(op.array, A.shape[1], k, p, q, seed, comm, GpuBackend(),
                                          amax=amax, sketch=sketch)
                torch.cuda.current_stream().synchronize()
                out[r] = {"U": res.U.cpu().numpy(), "Q": res.Q.cpu().numpy(),
                          "sigma": res.sigma.cpu().numpy(), "V": res.V.cpu().numpy(),
                          "est": res.est}
        except BaseException as e:  # pragma: no cover - reported below
            errs.append(e)
            shared["bar"].abort()

    ths = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    return out


def _check(A, outs, k, p, q, seed, s_tol, est_tol, sketch="gauss"):
    basis, f, est = orc.rsvd(A, k, p, q, seed, sketch=sketch)
    for key in ("sigma", "V"):
        assert np.array_equal(outs[0][key], outs[1][key]), key
    assert outs[0]["est"] == outs[1]["est"]
    Q = np.vstack([o["Q"] for o in outs])
    U = np.vstack([o["U"] for o in outs])
    S = outs[0]["sigma"]
    assert Q.shape[1] == basis.Q.shape[1]
    nq = Q.shape[1]
    assert np.linalg.norm(Q.conj().T.astype(np.complex128) @ Q - np.eye(nq)) < 100 * nq * s_tol
    assert np.max(np.abs(S - f.sigma) / f.sigma[0]) < s_tol
    assert abs(outs[0]["est"] - est) <= est_tol * est + 1e-12 * f.sigma[0]
    A_hat = (U * S) @ outs[0]["V"].conj().T
    assert np.linalg.norm(A - A_hat, 2) <= 10 * max(est, 1e-12 * f.sigma[0])


def _decay(m, n, rate, seed=3):
    import workloads
    return workloads.synthetic_explicit(m, n, np.exp(-np.arange(n) / rate), seed)[0]


def test_threads_f64_subspace_iteration():
    A = _decay(1100, 420, 12.0)
    outs = _run_threads(A, [0, 517, 1100], 20, 10, 2, 11)
    _check(A, outs, 20, 10, 2, 11, 1e-10, 1e-8)


def test_threads_f64_rank_deficient_cgs2_fallback():
    rng = np.random.default_rng(4)
    A = rng.standard_normal((700, 6)) @ rng.standard_normal((6, 300))
    outs = _run_threads(A, [0, 333, 700], 10, 6, 1, 2)
    _check(A, outs, 10, 6, 1, 2, 1e-10, 1e-6)


def test_threads_c128_srft():
    rng = np.random.default_rng(5)
    m, n = 640, 256
    U, _ = np.linalg.qr(rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    A = (U * np.exp(-np.arange(n) / 10.0)) @ V.conj().T
    outs = _run_threads(A, [0, 300, 640], 16, 8, 0, 9, sketch="srft")
    _check(A, outs, 16, 8, 0, 9, 1e-10, 1e-8, sketch="srft")


def test_threads_f32_power():
    import torch
    A = _decay(4096, 1024, 20.0).astype(np.float32)
    outs = _run_threads(A, [0, 2048, 4096], 32, 16, 1, 7, dtype=torch.float32)
    _check(A.astype(np.float64), outs, 32, 16, 1, 7, 1e-4, 1e-2)


def test_nccl_world1_public_entry():
    import torch
    import torch.distributed as dist
    from paper_0909_4061_b200.dist import sharded_randomized_svd
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        A = _decay(900, 300, 9.0)
        U, S, V, est = sharded_randomized_svd(A, 20, 10, 1, seed=4)
        _, f, est_ref = orc.rsvd(A, 20, 10, 1, 4)
        assert np.max(np.abs(S - f.sigma) / f.sigma[0]) < 1e-10
        assert abs(est - est_ref) <= 1e-8 * est_ref
        assert isinstance(U, np.ndarray) and U.shape == (900, 30)
        bad = A.copy()
        bad[3, 4] = np.nan
        with pytest.raises(ValueError):
            sharded_randomized_svd(bad, 5, 5, 0)
    finally:
        dist.destroy_process_group()


def test_nccl_world1_sparse_operator_path():
    """dist_randomized_svd_operator (config 5's sharded path) over NCCL with
    one rank: the same factors as the oracle on S + L R^T."""
    import scipy.sparse as sp
    import torch
    import torch.distributed as dist
    import paper_0909_4061_b200 as lr
    from paper_0909_4061_b200.dist import Comm, GpuBackend, dist_randomized_svd_operator
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        g = np.random.default_rng(41)
        n = 5000
        cols = g.integers(0, n, size=(n, 12))
        S = sp.csr_matrix((g.standard_normal(n * 12), (np.repeat(np.arange(n), 12), cols.ravel())),
                          shape=(n, n))
        S.sum_duplicates()
        L, R = 10 * g.standard_normal((n, 4)), 10 * g.standard_normal((n, 4))
        op = lr.CudaCsrOperator(S, L, R)
        res = dist_randomized_svd_operator(op, n, 6, 4, 2, 5, Comm(), GpuBackend())
        _, f, est = orc.rsvd(orc.SparsePlusLowRank(S, L, R), 6, 4, 2, 5)
        sig = res.sigma.cpu().numpy()
        assert np.max(np.abs(sig - f.sigma) / f.sigma[0]) < 1e-10
        assert abs(res.est - est) <= 1e-8 * est
        V = res.V.cpu().numpy()
        assert np.linalg.norm(V[:, 0] - f.V[:, 0]) < 1e-7
    finally:
        dist.destroy_process_group()


def test_c_abi_comm_world1():
    """The C ABI's own collectives (lr_comm_*), for callers without
    torch.distributed: a one-rank NCCL communicator on the handle;
    lr_orth_sharded equals lr_orth_fast bit for bit, the all-reduce is the
    identity."""
    import ctypes
    import torch
    from paper_0909_4061_b200 import _lib
    idbuf = ctypes.create_string_buffer(128)
    _lib.call("lr_comm_unique_id", ctypes.cast(idbuf, ctypes.c_void_p))
    h = _lib.handle()
    _lib.call("lr_comm_init", h, ctypes.cast(idbuf, ctypes.c_void_p), 1, 0)
    try:
        g = torch.Generator(device="cuda").manual_seed(3)
        Y = torch.randn(5000, 40, dtype=torch.float64, device="cuda", generator=g)
        Q1 = torch.empty_like(Y)
        Q2 = torch.empty_like(Y)
        st = torch.zeros(2, dtype=torch.int32, device="cuda")
        _lib.call("lr_orth_sharded", h, _lib.F64, 5000, 40, _lib.ptr(Y), 40, _lib.ptr(Q1), 40,
                  1e-10, _lib.ptr(st[0:1]))
        _lib.call("lr_orth_fast", h, _lib.F64, 5000, 40, _lib.ptr(Y), 40, _lib.ptr(Q2), 40,
                  1e-10, _lib.ptr(st[1:2]))
        assert int(st.sum().item()) == 0
        assert torch.equal(Q1, Q2)
        b = torch.arange(10, dtype=torch.float64, device="cuda")
        _lib.call("lr_comm_allreduce", h, _lib.F64, 10, _lib.ptr(b))
        torch.cuda.synchronize()
        assert torch.equal(b, torch.arange(10, dtype=torch.float64, device="cuda"))
    finally:
        _lib.call("lr_comm_destroy", h)
