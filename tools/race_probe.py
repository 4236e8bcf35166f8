"""Development probe: repeat the small kernels on identical inputs and report
any run-to-run difference (nondeterminism = a race)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_0909_4061_b200 as m
from paper_0909_4061_b200 import core, _lib
g = np.random.default_rng(5)
for cplx in (False, True):
    for ell in (40, 110, 120, 200):
        if cplx and ell > 140:
            continue
        Y = g.standard_normal((3 * ell, ell)) + (1j * g.standard_normal((3 * ell, ell)) if cplx else 0)
        Yd = torch.from_numpy(Y).cuda()
        G = (Yd.conj().T @ Yd).contiguous()
        code = _lib.C128 if cplx else _lib.F64
        outs = []
        for rep in range(30):
            P, R = torch.empty_like(G), torch.empty_like(G)
            info = torch.zeros(4, dtype=torch.int32, device="cuda")
            _lib.call("lr_chol_drop", _lib.handle(), code, ell, _lib.ptr(G), 1e-10, 4 * ell * 1.1e-16,
                      0.0, _lib.ptr(P), _lib.ptr(R), _lib.ptr(info))
            outs.append((P.cpu().numpy(), R.cpu().numpy()))
        dP = max(np.abs(o[0] - outs[0][0]).max() for o in outs)
        dR = max(np.abs(o[1] - outs[0][1]).max() for o in outs)
        print(f"chol ell={ell} cplx={cplx}: max run-to-run |dP| {dP:.2e} |dR| {dR:.2e}", flush=True)
        Z = torch.from_numpy(Y).cuda().contiguous()
        outs = []
        for rep in range(10):
            U, S, V = core.small_svd_from_adjoint(Z.clone())
            outs.append((S.cpu().numpy(), U.cpu().numpy()))
        dS = max(np.abs(o[0] - outs[0][0]).max() for o in outs)
        dU = max(np.abs(o[1] - outs[0][1]).max() for o in outs)
        print(f"  small_svd: |dS| {dS:.2e} |dU| {dU:.2e}", flush=True)
