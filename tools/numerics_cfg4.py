"""Offline numerics study for config 4 (fp32, ell=256, q=1) at reduced rows.

Emulates candidate tensor-core arithmetic schemes for the passes over A and
for the m-side orthonormalization, and compares the singular values of the
resulting randomized SVD with an fp64 run on the same A and Omega.  This is
a design-time tool ("decide the scheme by measured
parity"); results are recorded in DESIGN.md.

Usage: python tools/numerics_cfg4.py [m]
"""
import sys
import time

import numpy as np

m = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
n, ell, q, k = 4096, 256, 1, 200
rng = np.random.default_rng(4)


def haar(r, c):
    g = rng.standard_normal((r, c))
    qq, rr = np.linalg.qr(g)
    return qq * np.where(np.diag(rr) >= 0, 1.0, -1.0)


t0 = time.time()
U = haar(m, n)
V = haar(n, n)
s = np.where(np.arange(1, n + 1) <= 200, 0.9 ** np.arange(n), 1e-6)
A64 = ((U * s) @ V.T)
A32 = A64.astype(np.float32)
A64 = A32.astype(np.float64)  # the stored matrix is fp32; the oracle upcasts it
del U, V
Om = rng.standard_normal((n, ell))
print(f"built A {m}x{n} in {time.time()-t0:.1f}s", flush=True)


def tf32(x):
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return b.view(np.float32)


def bf16(x):
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)


def split(x, kind):
    x = np.asarray(x, dtype=np.float32)
    if kind == "tf32":
        h = tf32(x)
        return h, tf32(x - h)
    h = bf16(x)
    return h, bf16(x - h)


def mm(kind, L, R):
    """L @ R for fp32 operands under the named arithmetic scheme."""
    if kind == "f64":
        return L.astype(np.float64) @ R.astype(np.float64)
    L = np.asarray(L, np.float32)
    R = np.asarray(R, np.float32)
    if kind == "f32":
        return L @ R
    if kind == "tf32x1":
        return tf32(L) @ tf32(R)
    if kind in ("tf32x3", "bf16x3"):
        base = "tf32" if kind == "tf32x3" else "bf16"
        L1, L2 = split(L, base)
        R1, R2 = split(R, base)
        return (L2 @ R1 + L1 @ R2) + L1 @ R1
    if kind == "fp16x3":
        def sc(M):
            e = np.floor(np.log2(np.abs(M).max())) if np.abs(M).max() > 0 else 0
            return np.float32(2.0 ** (14 - e))
        sL, sR = sc(L), sc(R)
        Ls, Rs = L * sL, R * sR
        L1 = Ls.astype(np.float16).astype(np.float32); L2 = (Ls - L1).astype(np.float16).astype(np.float32)
        R1 = Rs.astype(np.float16).astype(np.float32); R2 = (Rs - R1).astype(np.float16).astype(np.float32)
        return ((L2 @ R1 + L1 @ R2) + L1 @ R1) / (sL * sR)
    if kind == "Aexact_Xbf2":
        R1, R2 = split(R, "bf16")
        return L @ (R1 + R2)
    if kind == "Abf2_Xexact":
        L1, L2 = split(L, "bf16")
        return (L1 + L2) @ R
    if kind == "bf16x6":
        L1, L2 = split(L, "bf16"); L3 = bf16(L - L1 - L2)
        R1, R2 = split(R, "bf16"); R3 = bf16(R - R1 - R2)
        return ((L3 @ R1 + L2 @ R2 + L1 @ R3) + (L2 @ R1 + L1 @ R2)) + L1 @ R1
    raise ValueError(kind)


def qr_pos(Y):
    Q, R = np.linalg.qr(Y)
    return Q * np.where(np.diag(R) >= 0, 1.0, -1.0)


def orth(Y, kind):
    if kind == "f64":
        return qr_pos(Y.astype(np.float64))
    Y = Y.astype(np.float32)
    if kind == "cholqr2_g64":
        Q = Y
        for _ in range(2):
            Q64 = Q.astype(np.float64)
            G = Q64.T @ Q64
            R = np.linalg.cholesky(G).T
            Q = np.linalg.solve(R.T, Q64.T).T.astype(np.float32)
        return Q
    if kind == "scholqr3_g32":
        Q = Y
        G = (Q.T @ Q).astype(np.float64)
        sh = 11 * (m * ell + ell * (ell + 1)) * 2.0**-24 * np.trace(G)
        sh = min(sh, 1e-3 * np.trace(G) / ell)
        R = np.linalg.cholesky(G + sh * np.eye(ell)).T
        Q = np.linalg.solve(R.T, Q.astype(np.float64).T).T.astype(np.float32)
        for _ in range(2):
            G = (Q.T @ Q).astype(np.float64)
            R = np.linalg.cholesky(G).T
            Q = np.linalg.solve(R.T, Q.astype(np.float64).T).T.astype(np.float32)
        return Q
    raise ValueError(kind)


def rsvd(gk, ok):
    first = gk
    if gk.startswith("mixed"):   # pass 1 bf16x3 (no A scale needed), rest fp16x3
        first, gk = "bf16x3", "fp16x3"
    Y = mm(first, A32, Om)
    Q = orth(Y, ok)
    Yt = mm(gk, A32.T, Q)
    Qt = orth(Yt, "f64" if ok == "f64" else "cholqr2_g64")
    Y = mm(gk, A32, Qt)
    Q = orth(Y, ok)
    Z = mm(gk, A32.T, Q)  # B^T = A^T Q  (n x ell)
    return np.linalg.svd(Z.astype(np.float64), compute_uv=False)


ref = rsvd("f64", "f64")
print("fp64 oracle done", flush=True)
SCHEMES = [("f32", "cholqr2_g64"), ("f32", "scholqr3_g32"), ("tf32x1", "cholqr2_g64"),
           ("bf16x3", "cholqr2_g64"), ("bf16x3", "scholqr3_g32"), ("tf32x3", "cholqr2_g64"),
           ("bf16x6", "cholqr2_g64"), ("fp16x3", "cholqr2_g64"), ("fp16x3", "scholqr3_g32"),
           ("Aexact_Xbf2", "cholqr2_g64"), ("Abf2_Xexact", "cholqr2_g64"),
           ("mixed", "cholqr2_g64")]
sel = sys.argv[2].split(",") if len(sys.argv) > 2 else None
for gk, ok in SCHEMES:
    if sel and f"{gk}/{ok}" not in sel and gk not in sel:
        continue
    t0 = time.time()
    try:
        sv = rsvd(gk, ok)
    except np.linalg.LinAlgError as e:
        print(f"{gk:8s} {ok:14s} FAILED: {e}", flush=True)
        continue
    rel = np.abs(sv - ref) / ref
    bad = np.nonzero(rel[:k] > 1e-4)[0]
    first = int(bad[0]) + 1 if bad.size else None
    print(f"{gk:8s} {ok:14s} first j>1e-4: {first}  max rel(top100)={rel[:100].max():.2e} "
          f"normwise={np.abs(sv-ref).max()/ref[0]:.2e}  ({time.time()-t0:.0f}s)", flush=True)
