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
