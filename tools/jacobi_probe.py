"""Development probe: one small SVD at a given ell (mixed, non-graded B) --
for ncu captures of the Jacobi kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0909_4061_b200 import core

ell, nc = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(0)
W = np.linalg.qr(rng.standard_normal((ell, ell)))[0]
V = np.linalg.qr(rng.standard_normal((nc, ell)))[0]
B = (W * (np.arange(1, ell + 1) ** -0.5)) @ V.T
Z = torch.from_numpy(B.T.copy()).cuda()
for _ in range(2):
    core.small_svd_from_adjoint(Z.clone())
torch.cuda.synchronize()
