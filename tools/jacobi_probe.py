"""Development probe: cluster Jacobi kernel time and sweep count (lr_jacobi_svd
path through the small SVD) at ell = 256 real / 120 complex / 110 real, for
variant libraries (LOWRANK_B200_LIB) built with -DLR_JAC_NOSUB / -DLR_JAC_NOXCHG."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0909_4061_b200 import core

rng = np.random.default_rng(0)
for ell, ncols, cplx in [(256, 4096, False), (120, 8192, True), (110, 8192, False)]:
    W = np.linalg.qr(rng.standard_normal((ell, ell)))[0]
    V = np.linalg.qr(rng.standard_normal((ncols, ell)))[0]
    B = (W * (np.arange(1, ell + 1) ** -0.5)) @ V.T
    if cplx:
        B = B + 1j * ((np.linalg.qr(rng.standard_normal((ell, ell)))[0] * 0.5) @ V.T)
    Z = torch.from_numpy(B).cuda().conj().T.contiguous()
    status = torch.zeros(1, dtype=torch.int32, device="cuda")

    def svd():
        with core.speculate(status):
            return core.small_svd_from_adjoint(Z.clone())

    for _ in range(2):
        svd()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        svd()
    e.record()
    torch.cuda.synchronize()
    print(f"ell={ell} cplx={cplx}: small_svd {s.elapsed_time(e) / 5 * 1e3:.1f} us, flags {int(status.item())}", flush=True)
