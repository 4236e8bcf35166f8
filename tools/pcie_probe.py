"""Development probe: host<->device copy rates of this box (pinned, one large
copy vs the 64 MiB row chunks of the streamed upload) and the split of one
config-4-shaped end-to-end call (upload / compute / download)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_0909_4061_b200 as lr

GB = 1e9


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


m, n = int(os.environ.get("M", 1 << 19)), 4096
host = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
host.normal_()
dev = torch.empty((m, n), dtype=torch.float32, device="cuda")
nbytes = host.numel() * 4
t = wall(lambda: dev.copy_(host, non_blocking=True))
print(f"H2D one copy {nbytes / GB:.2f} GB: {nbytes / t / GB:.1f} GB/s")
side = torch.cuda.Stream()
for chunk_mib in (16, 64, 256):
    rows = (chunk_mib << 20) // (n * 4)

    def chunked():
        with torch.cuda.stream(side):
            for r in range(0, m, rows):
                dev[r:r + rows].copy_(host[r:r + rows], non_blocking=True)
        torch.cuda.current_stream().wait_stream(side)

    t = wall(chunked)
    print(f"H2D {chunk_mib} MiB chunks: {nbytes / t / GB:.1f} GB/s")
back = torch.empty((m // 4, n), dtype=torch.float32, pin_memory=True)
t = wall(lambda: back.copy_(dev[: m // 4], non_blocking=True))
print(f"D2H one copy {back.numel() * 4 / GB:.2f} GB: {back.numel() * 4 / t / GB:.1f} GB/s")

# one end-to-end call, split
for _ in range(2):
    lr.randomized_svd(host, 200, 56, 1, 4, estimate=False)
torch.cuda.synchronize()
t0 = time.perf_counter()
op = lr.DenseOperator(host)
_ = op.array
torch.cuda.synchronize()
t1 = time.perf_counter()
b, f, _ = lr.randomized_svd(op, 200, 56, 1, 4, estimate=False)
torch.cuda.synchronize()
t2 = time.perf_counter()
t3 = time.perf_counter()
b, f, _ = lr.randomized_svd(host, 200, 56, 1, 4, estimate=False)
t4 = time.perf_counter()
print(f"upload+check {1e3 * (t1 - t0):.1f} ms ({nbytes / (t1 - t0) / GB:.1f} GB/s), "
      f"svd on the resident operator (host outputs) {1e3 * (t2 - t1):.1f} ms, whole call {1e3 * (t4 - t3):.1f} ms")
