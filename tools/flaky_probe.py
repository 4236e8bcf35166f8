import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_0909_4061_b200.core import DenseOperator
def rand(shape, dtype, seed):
    g = np.random.default_rng(seed); a = g.standard_normal(shape)
    if np.dtype(dtype).kind == "c": a = a + 1j * g.standard_normal(shape)
    return a.astype(dtype)
m, n, ell = 2048, 2048, 30
A = rand((m, n), np.complex128, m + n); X = rand((n, ell), np.complex128, ell); W = rand((m, ell), np.complex128, ell+1)
op = DenseOperator(A)
ref = A @ X; refz = A.conj().T @ W
for i in range(8):
    Y = op.apply(X); Z = op.apply_adjoint(W)
    ey = np.abs(Y - ref).max(); ez = np.abs(Z - refz).max()
    bad = np.argwhere(np.abs(Y - ref) > 1e-9)
    print(i, f"{ey:.2e} {ez:.2e}", bad[:5].tolist(), len(bad))
