"""Development probe: random tall fp32 panels through the sketch-preconditioned
orthonormalization -- a run with status 0 must be orthonormal at the fp32 level
and span the panel; flagged runs are counted (they rerun on the exact path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0909_4061_b200 import core

rng = np.random.default_rng(int(os.environ.get("SEED", 0)))
flagged = bad = 0
N = int(os.environ.get("N", 40))
for it in range(N):
    m = int(rng.integers(65536, 300000))
    ell = int(rng.choice([16, 20, 32, 48, 64, 100, 128, 200, 256]))
    ell = ell - ell % 4                       # fp32 rows 16-byte aligned
    kappa = 10.0 ** rng.uniform(0, 7.5)
    kind = rng.choice(["haar", "heavy", "sparse_rows", "dup_scale"])
    g = torch.Generator(device="cuda").manual_seed(it)
    U = torch.randn(m, ell, device="cuda", dtype=torch.float64, generator=g)
    if kind == "heavy":
        U[:: max(1, m // 37)] *= 1e3
    elif kind == "sparse_rows":               # most rows zero: a coherent range
        mask = torch.rand(m, device="cuda", generator=g) < 0.01
        U = U * mask[:, None]
    U, _ = torch.linalg.qr(U)
    W, _ = torch.linalg.qr(torch.randn(ell, ell, device="cuda", dtype=torch.float64, generator=g))
    s = torch.logspace(0, -float(np.log10(kappa)), ell, device="cuda", dtype=torch.float64)
    Y = ((U * s) @ W.T)
    if kind == "dup_scale":
        Y = Y * float(10.0 ** rng.uniform(-20, 20))
    Y = Y.float().contiguous()
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    with core.speculate(status):
        Q = core.orth_dev(Y)
    torch.cuda.synchronize()
    st = int(status.item())
    if st:
        flagged += 1
        print(f"[{it}] m={m} ell={ell} kappa={kappa:.1e} {kind}: flagged {st}", flush=True)
        continue
    Qd, Yd = Q.double(), Y.double()
    orth = (Qd.T @ Qd - torch.eye(ell, device="cuda", dtype=torch.float64)).abs().max().item()
    R = Qd.T @ Yd
    span = (torch.linalg.norm(Yd - Qd @ R) / torch.linalg.norm(Yd)).item()
    # span residual is limited by fp32 rounding of Y itself times the growth of R^{-1}
    ok = orth <= 5e-6 and span <= 1e-4
    if not ok:
        bad += 1
    print(f"[{it}] m={m} ell={ell} kappa={kappa:.1e} {kind}: orth {orth:.1e} span {span:.1e} {'OK' if ok else 'BAD'}",
          flush=True)
    del U, Y, Q, Qd, Yd
print(f"{N} panels: {flagged} flagged, {bad} bad")
