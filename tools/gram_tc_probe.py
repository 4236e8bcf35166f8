"""Development probe: error of the tensor-core Gram (lr_gram_tc) on a panel
with kappa ~ 3 (what the sketch-preconditioned first pass leaves), against the
fp64 Gram: size of the error, its correlation with G (a coherent truncation
bias shows as a negative regression slope), and its spectral norm."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0909_4061_b200 import _lib

m, ell = 1 << 20, 256
g = torch.Generator(device="cuda").manual_seed(3)
U, _ = torch.linalg.qr(torch.randn(m, ell, device="cuda", dtype=torch.float64, generator=g))
M = torch.randn(ell, ell, device="cuda", dtype=torch.float64, generator=g)
W1, _ = torch.linalg.qr(M)
s = torch.linspace(0.6, 1.8, ell, device="cuda", dtype=torch.float64)
Y = ((U * s) @ W1.T).float().contiguous()
Yd = Y.double()
Gx = Yd.T @ Yd
G = torch.empty(ell, ell, dtype=torch.float64, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
_lib.call("lr_gram_tc", _lib.handle(0), m, ell, _lib.ptr(Y), ell, _lib.ptr(G), 12, _lib.ptr(st))
torch.cuda.synchronize()
G = torch.triu(G) + torch.triu(G, 1).T
E = G - Gx
off = ~torch.eye(ell, dtype=torch.bool, device="cuda")
slope = (E[off] * Gx[off]).sum() / (Gx[off] ** 2).sum()
print(f"status {int(st.item())} max|E| {E.abs().max().item():.3e} max|E_off| {E[off].abs().max().item():.3e} "
      f"rms off G {Gx[off].pow(2).mean().sqrt().item():.3e} rms off E {E[off].pow(2).mean().sqrt().item():.3e} "
      f"slope E~G {slope.item():.3e} ||E||2 {torch.linalg.matrix_norm(E, 2).item():.3e} "
      f"||E - slope G_off||2 {torch.linalg.matrix_norm(E - slope * Gx * off, 2).item():.3e}")
