"""One config-4-shaped call of each panel kernel (m = 2^20, ell = 256): the
m-side apply Y P (gemm_f32_pair_kernel via lr_gemm_scaled, K = 256), the
tcgen05 Gram (lr_gram_tc) and an A^T Y pass operand split
(split_transpose_kernel) -- for ncu --set full captures (profiles/)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0909_4061_b200 import _lib, core  # noqa: E402

m, ell = 1 << 20, 256
g = torch.Generator(device="cuda").manual_seed(0)
Y = torch.randn(m, ell, device="cuda", generator=g) / 1024
P = torch.randn(ell, ell, device="cuda", generator=g)
Q = torch.empty(m, ell, device="cuda")
G = torch.empty(ell, ell, dtype=torch.float64, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
A = torch.randn(m, 64, device="cuda", generator=g)
Z = torch.empty(64, ell, device="cuda")
h = _lib.handle()
for _ in range(3):
    _lib.call("lr_gemm_scaled", h, _lib.F32, _lib.OP_N, m, ell, ell, _lib.ptr(Y), ell, -1.0,
              _lib.ptr(P), ell, _lib.ptr(Q), ell)
    _lib.call("lr_gram_tc", h, m, ell, _lib.ptr(Y), ell, _lib.ptr(G), 12, _lib.ptr(st))
    core._pass(A, Y, Z, True, float(A.abs().max()))
torch.cuda.synchronize()
