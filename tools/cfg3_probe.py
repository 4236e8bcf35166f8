"""Development probe: cfg3 estimator pass under SIMT vs tcgen05 arithmetic."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_0909_4061_b200 as lr
import workloads
from paper_0909_4061_b200 import core

A = workloads.build_cfg3()
op = lr.DenseOperator(A)
print("amax", op.amax)
W = torch.from_numpy(lr.rng_for(16, 0x70726F62).standard_normal((8192, 10))).cuda().to(torch.complex64)
ref = torch.from_numpy(A.astype(np.complex128)).cuda() @ W.to(torch.complex128)
for mode in (lr._lib.F32_SIMT, lr._lib.F32_SPLIT3):
    lr._lib.set_f32_mode(mode)
    Z = op.apply(W)
    err = (Z.to(torch.complex128) - ref).abs()
    print("mode", mode, "max abs err", err.max().item(), "max |ref|", ref.abs().max().item(),
          "rel", err.max().item() / ref.abs().max().item(), flush=True)
    b, f, est = lr.randomized_svd(op, 50, 70, 0, 3, sketch="srft")
    print("  est", est, "sigma0", float(f.sigma[0]))
