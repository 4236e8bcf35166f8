"""Test-only backend for paper_0909_4061_b200.dist: the same primitives as
GpuBackend computed with torch CPU tensors / the numpy oracle, so the
row-sharded host logic (collective order, rank decisions, fallbacks) can be
exercised over gloo with world_size > 1 in a container without a GPU.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import lowrank_oracle as orc


def _np(t):
    return t.detach().numpy()


class TorchCpuBackend:
    def __init__(self):
        self.torch = torch

    # --- a row-block operator given as (S_r scipy CSR, L_r, R): S_r + L_r R^T
    def op_n(self, op, X):
        S, L, R = op
        x = _np(X)
        return torch.from_numpy(np.asarray(S @ x + L @ (R.T @ x)))

    def op_t(self, op, Y):
        S, L, R = op
        y = _np(Y)
        return torch.from_numpy(np.asarray(S.T @ y + R @ (L.T @ y)))

    def like(self, op):
        return torch.empty(0, dtype=torch.float64)

    def pass_n(self, A, X, amax=None):
        return A @ X

    def pass_t(self, A, Y, amax=None):
        return A.conj().T @ Y

    def gram(self, Y):
        return (Y.conj().T @ Y).contiguous()

    def chol(self, G, drop_tol, unres_rel, shift_coef):
        """Cholesky with column deletion -- the numpy restatement of the
        lr_chol_drop contract (csrc/chol.cu): pivot d_j = G_jj + shift -
        sum_{i kept < j} |r_ij|^2; kept iff finite and > tol^2 tr(G)."""
        g = _np(G)
        n = g.shape[0]
        tr = float(np.real(np.trace(g)))
        thr2 = drop_tol * drop_tol * tr
        shift = shift_coef * tr
        R = np.zeros_like(g)
        kept, unres, bad = [], 0, 0
        for j in range(n):
            for a, i in enumerate(kept):
                s = g[i, j] - sum(np.conj(R[l, i]) * R[l, j] for l in kept[:a])
                R[i, j] = s / R[i, i]
            d = float(np.real(g[j, j])) + shift - sum(abs(R[i, j]) ** 2 for i in kept)
            if np.isfinite(d) and d > thr2 and d > 0.0:
                R[j, j] = np.sqrt(d)
                if d <= unres_rel * (float(np.real(g[j, j])) + shift):
                    unres += 1
                kept.append(j)
            else:
                if not np.isfinite(d):
                    bad += 1
                R[:, j] = 0
        P = np.zeros_like(g)
        if kept:
            Rk = R[np.ix_(kept, kept)]
            P[np.ix_(kept, list(range(len(kept))))] = np.linalg.inv(Rk)
        return torch.from_numpy(P), torch.from_numpy(R), len(kept), unres, bad

    def chol_fast(self, G, drop_tol, unres_rel, near_thr, status):
        P, _, rank, unres, bad = self.chol(G, drop_tol, unres_rel, 0.0)
        bits = (1 if unres else 0) | (2 if rank < G.shape[0] else 0) | (4 if bad else 0)
        status |= bits
        return P

    def new_status(self, like):
        return torch.zeros(1, dtype=torch.int32)

    def status_value(self, status):
        return int(status.item())

    def speculate(self, status):
        import contextlib
        return contextlib.nullcontext()

    def apply(self, Y, P, ncols):
        return Y @ P[:, :ncols].to(Y.dtype)

    def matmul(self, A, B):
        return A @ B

    def adj_matmul(self, A, B):
        return A.conj().T @ B

    def sub_(self, Z, T):
        Z -= T
        return Z

    def colsumsq(self, Z):
        return (Z.abs() ** 2).sum(dim=0).to(torch.float64)

    def small_svd(self, Z):
        f = orc.small_svd(_np(Z).conj().T)
        return torch.from_numpy(f.U), torch.from_numpy(f.sigma), torch.from_numpy(f.V)

    def orth_local(self, Z):
        return torch.from_numpy(orc.orthonormalize_double_gs(_np(Z)))

    def gaussian(self, n, ell, seed, stream, like):
        g = orc.rng_for(seed, stream).standard_normal((n, ell))
        return torch.from_numpy(g).to(like.dtype)

    def zeros_like_rows(self, Y, ncols):
        return torch.zeros((Y.shape[0], ncols), dtype=Y.dtype)

    def zeros_rows(self, rows, ncols, like):
        return torch.zeros((rows, ncols), dtype=like.dtype)

    def empty_sigma(self, like):
        return torch.zeros(0, dtype=torch.float64)

    def trace(self, G):
        return float(torch.diagonal(G).real.sum())

    def column(self, Y, j):
        return Y[:, j:j + 1].clone()

    def set_column(self, Q, j, w, inv):
        Q[:, j:j + 1] = w * inv

    def to_scalar(self, t):
        return float(t.max())
