import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_0909_4061_b200 as m
from paper_0909_4061_b200 import core, factor
from oracle import lowrank_oracle as O
g = np.random.default_rng(5)
n, ell = 3000, 40
X = g.standard_normal((n, n)) + 1j * g.standard_normal((n, n))
U = np.linalg.qr(X)[0][:, :200]
lam0 = np.exp(-np.arange(200) / 15.0) * np.where(np.arange(200) % 3 == 1, -1.0, 1.0)
A = ((U * lam0) @ U.conj().T).astype(np.complex128)
A = 0.5 * (A + A.conj().T)
Q0 = m.randomized_range_finder(A, ell, seed=3).Q
fo = O.direct_eig_hermitian(A, Q0)
for it in range(25):
    Q = m.randomized_range_finder(A, ell, seed=3).Q
    dq = np.abs(Q - Q0).max()
    op = m.DenseOperator(A)
    Qd = core.to_device(Q, torch.complex128)
    Y = core.apply_dev(op, Qd)
    B = torch.empty((ell, ell), dtype=torch.complex128, device="cuda")
    core.gemm(Qd, Y, B, adjoint=True)
    Bh = Q.conj().T @ (A @ Q)
    dB = np.abs(B.cpu().numpy() - Bh).max()
    V, lam = core.small_eig_hermitian_dev(B)
    lr_, _ = np.linalg.eigh(0.5 * (Bh + Bh.conj().T)); o = np.lexsort((-lr_, -np.abs(lr_)))
    dl = np.abs(lam.cpu().numpy() - lr_[o]).max()
    f = m.direct_eig_hermitian(op, Q)
    df = np.abs(f.lam - fo.lam).max()
    Hs = Bh + 2 * np.linalg.norm(Bh) * np.eye(ell)
    fs = m.small_svd(Hs)
    ds = np.abs(fs.sigma - np.linalg.svd(Hs, compute_uv=False)).max()
    print(f"it {it}: dQ {dq:.1e} dB {dB:.1e} dlam {dl:.1e} dfull {df:.1e} dsvd {ds:.1e}", flush=True)
