"""Development probe: where one end-to-end config-4 call (pinned host A in,
host factors out) spends its wall time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_0909_4061_b200 as lr
from paper_0909_4061_b200 import core, factor

m, n = int(os.environ.get("M", 1 << 20)), 4096
host = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
host.normal_()


def once(split):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = lr.DenseOperator(host)
    if split:
        torch.cuda.synchronize()
    t1 = time.perf_counter()
    b, f, _ = lr.randomized_svd(op, 200, 56, 1, 4, estimate=False)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


for i in range(4):
    print("split: upload %.1f ms, svd+outputs %.1f ms" % tuple(1e3 * x for x in once(True)), flush=True)
for i in range(3):
    a, b = once(False)
    print("unsplit: ctor %.1f ms, rest %.1f ms, total %.1f" % (1e3 * a, 1e3 * b, 1e3 * (a + b)), flush=True)
# outputs only
op = lr.DenseOperator(host)
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b, f, _ = lr.randomized_svd(op, 200, 56, 1, 4, estimate=False)
    t1 = time.perf_counter()
    print("resident operator, host outputs: %.1f ms" % (1e3 * (t1 - t0)), flush=True)
dev = op.array
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b, f, _ = lr.randomized_svd(dev, 200, 56, 1, 4, estimate=False)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print("device in / device out: %.1f ms" % (1e3 * (t1 - t0)), flush=True)
