"""Measurement of the Hermitian Stage-B routes:
direct_eig_hermitian (factor.py:181-191) and eig_nystrom (factor.py:300-335)
on a cfg2-sized Hermitian input (n = 8192, fp64, ell = 110; H = U diag(s) U^T
with Haar U from the seeded generator, s_j = j^{-1/2} with alternating signs
for the eigen route, positive for Nystrom).  The basis comes from the device
range finder (not timed).  Device-resident inputs, CUDA events, L2 not
flushed (H is 512 MiB > L2).  The CPU oracle is timed on the same inputs.

    python tools/bench_stageb.py [--steps K] [--warmup W] [--n N] [--ell L]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_0909_4061_b200 as lr
from paper_0909_4061_b200 import factor


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--n", type=int, default=8192)
    p.add_argument("--ell", type=int, default=110)
    a = p.parse_args()
    n, ell = a.n, a.ell
    g = torch.Generator(device="cuda").manual_seed(17)
    U, _ = torch.linalg.qr(torch.randn(n, n, device="cuda", dtype=torch.float64, generator=g))
    s = torch.arange(1, n + 1, device="cuda", dtype=torch.float64) ** -0.5
    sign = torch.where(torch.arange(n, device="cuda") % 3 == 1, -1.0, 1.0).double()
    lines = []
    for route in ("eig", "nystrom"):
        lam = s * sign if route == "eig" else s
        H = (U * lam) @ U.T
        H = 0.5 * (H + H.T)
        op = lr.DenseOperator(H)
        Q = lr.randomized_range_finder(op, ell, seed=2).Q
        torch.cuda.synchronize()

        def step():
            if route == "eig":
                return lr.direct_eig_hermitian(op, Q)
            return lr.eig_nystrom(op, Q)[0]

        for _ in range(a.warmup):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            f = step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        passes = 3 if route == "eig" else 1      # probe x2 + B (eig); B1 (nystrom)
        abytes = H.numel() * 8
        from oracle import lowrank_oracle as O
        Hh, Qh = H.cpu().numpy(), Q.cpu().numpy()
        t0 = time.perf_counter()
        fo = O.direct_eig_hermitian(Hh, Qh) if route == "eig" else O.eig_nystrom(Hh, Qh)[0]
        t_cpu = time.perf_counter() - t0
        lam_dev = f.lam.cpu().numpy()
        err = float(np.abs(lam_dev - fo.lam).max() / np.abs(fo.lam).max())
        lines.append({"route": route, "n": n, "ell": ell, "ms_per_step": round(ms, 4),
                      "value": round(passes * abytes / (ms / 1e3) / 1e9, 2), "unit": "A-GB/s",
                      "passes": passes, "dtype": "f64", "steps": a.steps, "warmup": a.warmup,
                      "lam_rel_err_vs_oracle": err,
                      "cpu_baseline": {"seconds": round(t_cpu, 4), "kind": "port",
                                       "cores": os.cpu_count(),
                                       "sample": f"one {route} route by the oracle"}})
        print(json.dumps(lines[-1]), flush=True)
        del H, op


if __name__ == "__main__":
    main()
