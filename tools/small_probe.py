"""Development probe: time the latency-bound small kernels (Cholesky with
deletion, small SVD) at the BASELINE configs' ell, and check the small SVD
against numpy.  Run twice with LR_JACOBI=round to compare Jacobi variants."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_0909_4061_b200 as lr
from paper_0909_4061_b200 import _lib, core


def timeit(fn, reps=20):
    """Device time per call: the calls are captured in a CUDA graph so the
    host-side ctypes overhead does not leak into the number."""
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


rng = np.random.default_rng(0)
for ell, ncols, cplx in [(30, 2048, False), (48, 4096, False), (110, 8192, False), (120, 8192, True),
                         (64, 4096, True), (128, 4096, False), (256, 4096, False)]:
    dt = torch.complex128 if cplx else torch.float64
    if os.environ.get("MIXED"):
        # B = W diag(s) V^T with random orthogonal W: rows of B are not graded
        # (like B = Q^T A with a range basis Q from CholeskyQR)
        W = np.linalg.qr(rng.standard_normal((ell, ell)))[0]
        V = np.linalg.qr(rng.standard_normal((ncols, ell)))[0]
        B = (W * (np.arange(1, ell + 1) ** -0.5)) @ V.T
        if cplx:
            B = B + 1j * ((np.linalg.qr(rng.standard_normal((ell, ell)))[0] * 0.5) @ V.T)
    else:
        B = rng.standard_normal((ell, ncols)) * np.exp(-np.arange(ell) / 30.0)[:, None]
        if cplx:
            B = B + 1j * rng.standard_normal((ell, ncols)) * np.exp(-np.arange(ell) / 30.0)[:, None]
    Bd = torch.from_numpy(B).cuda()
    Z = Bd.conj().T.contiguous()
    G = (Z.conj().T @ Z).contiguous()
    P = torch.empty_like(G)
    R = torch.empty_like(G)
    info = torch.zeros(4, dtype=torch.int32, device="cuda")
    code = _lib.C128 if cplx else _lib.F64

    def chol():
        _lib.call("lr_chol_drop", _lib.handle(), code, ell, _lib.ptr(G), 1e-10, 4 * ell * 1.1e-16,
                  0.0, _lib.ptr(P), _lib.ptr(R), _lib.ptr(info))

    t_chol = timeit(chol)
    chol()
    Q = Z @ P
    orth = (Q.conj().T @ Q - torch.eye(ell, device="cuda", dtype=dt)).abs().max().item()

    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    Zc = Z.clone()

    def svd():
        Zc.copy_(Z)
        with core.speculate(status):
            return core.small_svd_from_adjoint(Zc)

    svd()
    t_svd = timeit(svd, reps=5)
    with core.speculate(status):
        U, S, V = core.small_svd_from_adjoint(Z.clone())
    torch.cuda.synchronize()
    s_ref = np.linalg.svd(B, compute_uv=False)
    err = np.max(np.abs(S.cpu().numpy() - s_ref)) / s_ref[0]
    print(f"ell={ell:4d} ncols={ncols} cplx={cplx}: chol {t_chol:8.1f} us (info {info.tolist()}, "
          f"|Q^H Q - I| {orth:.1e}) | small_svd {t_svd:8.1f} us, sigma err {err:.1e}, flags {int(status.item())}", flush=True)
