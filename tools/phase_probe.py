"""Development probe: Cholesky phase cycles (LR_CHOL_PROF=1) and Jacobi sweep
counts (LR_DEBUG_JACOBI=1) at the BASELINE configs' ell, eager (the debug
hooks synchronize, so no graph capture here)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0909_4061_b200 import _lib, core

rng = np.random.default_rng(0)
for ell, ncols, cplx in [(110, 8192, False), (120, 8192, True), (128, 4096, False), (256, 4096, False)]:
    dt = torch.complex128 if cplx else torch.float64
    B = rng.standard_normal((ell, ncols)) * np.exp(-np.arange(ell) / 30.0)[:, None]
    if cplx:
        B = B + 1j * rng.standard_normal((ell, ncols)) * np.exp(-np.arange(ell) / 30.0)[:, None]
    Z = torch.from_numpy(B).cuda().conj().T.contiguous()
    G = (Z.conj().T @ Z).contiguous()
    P, R = torch.empty_like(G), torch.empty_like(G)
    info = torch.zeros(4, dtype=torch.int32, device="cuda")
    code = _lib.C128 if cplx else _lib.F64
    print(f"--- ell={ell} cplx={cplx}", flush=True)
    for _ in range(2):
        _lib.call("lr_chol_drop", _lib.handle(), code, ell, _lib.ptr(G), 1e-10, 4 * ell * 1.1e-16,
                  0.0, _lib.ptr(P), _lib.ptr(R), _lib.ptr(info))
    torch.cuda.synchronize()
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(2):
        with core.speculate(status):
            core.small_svd_from_adjoint(Z.clone())
    torch.cuda.synchronize()
