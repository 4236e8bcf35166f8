import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pytest
sel = sys.argv[1] if len(sys.argv) > 1 else "chol or orth or small_svd"
pytest.main(["-q", "-m", "gpu", "-k", sel, "tests/test_gpu_kernels.py", "-p", "no:cacheprovider"])
import numpy as np, torch
import paper_0909_4061_b200 as m
from paper_0909_4061_b200 import core
from oracle import lowrank_oracle as O
g = np.random.default_rng(5)
n, ell = 3000, 40
X = g.standard_normal((n, n)) + 1j * g.standard_normal((n, n))
U = np.linalg.qr(X)[0][:, :200]
lam0 = np.exp(-np.arange(200) / 15.0) * np.where(np.arange(200) % 3 == 1, -1.0, 1.0)
A = ((U * lam0) @ U.conj().T).astype(np.complex128)
A = 0.5 * (A + A.conj().T)
Q = m.randomized_range_finder(A, ell, seed=3).Q
print("Q dtype", Q.dtype, "orth", np.abs(Q.conj().T @ Q - np.eye(ell)).max())
op = m.DenseOperator(A)
Qd = core.to_device(Q, torch.complex128)
Y = core.apply_dev(op, Qd)
print("Y err", np.abs(Y.cpu().numpy() - A @ Q).max())
B = torch.empty((ell, ell), dtype=torch.complex128, device="cuda")
core.gemm(Qd, Y, B, adjoint=True)
Bh = Q.conj().T @ (A @ Q)
print("B err", np.abs(B.cpu().numpy() - Bh).max())
V, lam = core.small_eig_hermitian_dev(B)
lr_, _ = np.linalg.eigh(0.5 * (Bh + Bh.conj().T)); o = np.lexsort((-lr_, -np.abs(lr_)))
print("lam err (dev B)", np.abs(lam.cpu().numpy() - lr_[o]).max())
Hs = Bh + 2 * np.linalg.norm(Bh) * np.eye(ell)
f = m.small_svd(Hs)
print("svd err", np.abs(f.sigma - np.linalg.svd(Hs, compute_uv=False)).max())
