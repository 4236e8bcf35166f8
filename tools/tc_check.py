"""Development check of the fp32 tcgen05 pass kernel: accuracy vs fp64 and
timing for A X / A^T Y at cfg4-like sizes.  Usage: python tools/tc_check.py [m]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_0909_4061_b200 as lr
from paper_0909_4061_b200 import core

m = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
n, ell = 4096, 256
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(m, n, device="cuda", generator=g, dtype=torch.float32) * 3e-3
X = torch.randn(n, ell, device="cuda", generator=g, dtype=torch.float32)
Yq = torch.linalg.qr(torch.randn(m, ell, device="cuda", dtype=torch.float64, generator=g))[0].float().contiguous()
op = lr.DenseOperator(A)
print("amax", op.amax, flush=True)
for name, X_, adj in (("A X", X, False), ("A^T Y", Yq, True)):
    out = torch.empty((n if adj else m, ell), device="cuda", dtype=torch.float32)
    core._pass(A, X_, out, adj, op.amax)
    ref = (A.double().T if adj else A.double()) @ X_.double()
    err = (out.double() - ref).abs().max().item() / ref.abs().max().item()
    simt = torch.empty_like(out)
    lr._lib.set_f32_mode(lr._lib.F32_SIMT)
    core._pass(A, X_, simt, adj, op.amax)
    lr._lib.set_f32_mode(lr._lib.F32_SPLIT3)
    err_simt = (simt.double() - ref).abs().max().item() / ref.abs().max().item()
    for _ in range(2):
        core._pass(A, X_, out, adj, op.amax)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        core._pass(A, X_, out, adj, op.amax)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    flops = 2 * m * n * ell
    print(f"{name}: rel err tc {err:.2e} (simt fp32 {err_simt:.2e}); {ms:.3f} ms; "
          f"{flops / ms / 1e9:.1f} TFLOP/s (algorithmic); A {A.numel() * 4 / ms / 1e6:.0f} GB/s",
          flush=True)
