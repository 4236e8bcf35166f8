"""One config-4-shaped pass of each fp32 kernel (A X and A^T Y, 2^20 x 4096,
ell = 256) for an ncu --set full capture (profiles/)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0909_4061_b200 import core  # noqa: E402

m, n, ell = 1 << 20, 4096, 256
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(m, n, device="cuda", generator=g)
X = torch.randn(n, ell, device="cuda", generator=g)
Yt = torch.randn(m, ell, device="cuda", generator=g) / 1024
Y = torch.empty(m, ell, device="cuda")
Z = torch.empty(n, ell, device="cuda")
amax = float(A.abs().max())
for _ in range(2):
    core._pass(A, X, Y, False, amax)
    core._pass(A, Yt, Z, True, amax)
torch.cuda.synchronize()
