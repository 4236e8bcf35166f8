"""Development probe: tcgen05 pass error vs K length / N / data."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_0909_4061_b200 as lr
from paper_0909_4061_b200 import core

g = torch.Generator(device="cuda").manual_seed(0)
for (M, K, N) in [(1536, 2048, 20), (8192, 2048, 20), (1536, 16384, 20), (8192, 16384, 20),
                  (8192, 16384, 256), (8192, 4096, 20), (256, 16384, 20), (128, 4096, 32),
                  (128, 8192, 32)]:
    A = torch.randn(M, K, device="cuda", generator=g)
    X = torch.randn(K, N, device="cuda", generator=g)
    op = lr.DenseOperator(A)
    Y = torch.empty(M, N, device="cuda")
    core._pass(A, X, Y, False, op.amax)
    ref = A.double() @ X.double()
    err = (Y.double() - ref).abs()
    rel = err.max().item() / ref.abs().max().item()
    bad = (err > 1e-3 * ref.abs().max()).nonzero()
    rows = sorted(set(bad[:, 0].tolist()))[:8] if bad.numel() else []
    cols = sorted(set(bad[:, 1].tolist()))[:8] if bad.numel() else []
    print(f"M={M} K={K} N={N}: rel {rel:.2e}, bad {bad.shape[0]} rows {rows} cols {cols}",
          flush=True)
