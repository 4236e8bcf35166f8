import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_0909_4061_b200 import _lib
ell = int(sys.argv[1])
Z = torch.randn(8192, ell, dtype=torch.float64, device="cuda")
G = (Z.T @ Z).contiguous(); P = torch.empty_like(G); R = torch.empty_like(G)
info = torch.zeros(4, dtype=torch.int32, device="cuda")
for _ in range(3):
    _lib.call("lr_chol_drop", _lib.handle(), _lib.F64, ell, _lib.ptr(G), 1e-10, 4*ell*1.1e-16, 0.0, _lib.ptr(P), _lib.ptr(R), _lib.ptr(info))
torch.cuda.synchronize(); print(info.tolist())
