"""Where the end-to-end (host buffers in / out) time of a randomized SVD goes.

    python tools/e2e_probe.py [config]

Prints the pinned H2D rate for A, the pageable / pinned D2H rate for the
factors, and the wall time of the public call with host input split into
upload + validation, the device step, and the output copies.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402
import paper_0909_4061_b200 as lr  # noqa: E402


def wall(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    cfg = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
    A = bench.build_input(cfg)
    nb = A.numel() * A.element_size()
    host = torch.empty(A.shape, dtype=A.dtype, pin_memory=True)
    host.copy_(A)
    dev = torch.empty_like(A)
    t = wall(lambda: dev.copy_(host, non_blocking=True))
    print(f"H2D pinned {nb / 2**30:.2f} GiB: {t * 1e3:.2f} ms = {nb / t / 1e9:.1f} GB/s")
    out = torch.empty((cfg.m, cfg.ell), dtype=A.dtype, device="cuda")
    ob = out.numel() * out.element_size()
    t = wall(lambda: out.cpu())
    print(f"D2H pageable {ob / 1e6:.1f} MB: {t * 1e3:.3f} ms = {ob / t / 1e9:.1f} GB/s")
    ph = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
    t = wall(lambda: ph.copy_(out, non_blocking=True))
    print(f"D2H pinned   {ob / 1e6:.1f} MB: {t * 1e3:.3f} ms = {ob / t / 1e9:.1f} GB/s")

    t = wall(lambda: lr.DenseOperator(host))
    print(f"DenseOperator(host) upload+validate: {t * 1e3:.2f} ms")
    op = lr.DenseOperator(A)

    def dev_step():
        return lr.randomized_svd(op, cfg.k, cfg.p, cfg.q, cfg.seed, sketch=cfg.sketch,
                                 estimate=False)
    dev_step()
    t = wall(dev_step)
    print(f"device step (graph replay): {t * 1e3:.2f} ms")

    def host_step():
        return lr.randomized_svd(host, cfg.k, cfg.p, cfg.q, cfg.seed, sketch=cfg.sketch,
                                 estimate=False)
    host_step()
    t = wall(host_step)
    print(f"host step (public API, e2e): {t * 1e3:.2f} ms")
    b, f, _ = dev_step()
    t = wall(lambda: (b.Q.cpu(), f.U.cpu(), f.sigma.cpu(), f.V.cpu()))
    print(f"output copies Q,U,S,V pageable: {t * 1e3:.2f} ms")


if __name__ == "__main__":
    main()
