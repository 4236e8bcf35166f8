"""Development probe: one lr_chol_drop launch at a given ell (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0909_4061_b200 import _lib

ell = int(sys.argv[1]) if len(sys.argv) > 1 else 110
cplx = len(sys.argv) > 2 and sys.argv[2] == "c"
g = np.random.default_rng(0)
Y = g.standard_normal((4 * ell, ell)) + (1j * g.standard_normal((4 * ell, ell)) if cplx else 0)
Yd = torch.from_numpy(Y).cuda()
G = (Yd.conj().T @ Yd).contiguous()
P, R = torch.empty_like(G), torch.empty_like(G)
info = torch.zeros(4, dtype=torch.int32, device="cuda")
for _ in range(3):
    _lib.call("lr_chol_drop", _lib.handle(), _lib.C128 if cplx else _lib.F64, ell, _lib.ptr(G),
              1e-10, 4 * ell * 1.1e-16, 0.0, _lib.ptr(P), _lib.ptr(R), _lib.ptr(info))
torch.cuda.synchronize()
print(info.tolist())
