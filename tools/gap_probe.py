"""Kernel timeline of one (graph-replayed) randomized-SVD step: busy time vs
span, i.e. how much of the step is launch gaps between dependent kernels.

    python tools/gap_probe.py [config]

Uses torch.profiler (CUPTI activity records: kernel start/end on the GPU
clock); the step is replayed as the bench does (CUDA graph after warm-up).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402
import paper_0909_4061_b200 as lr  # noqa: E402


def main():
    cfg = workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
    if cfg.idx == 5:
        op = lr.CudaCsrOperator(*workloads.build_cfg5())
    else:
        op = lr.DenseOperator(bench.build_input(cfg))

    def step():
        return lr.randomized_svd(op, cfg.k, cfg.p, cfg.q, cfg.seed, sketch=cfg.sketch,
                                 estimate=False)
    for _ in range(4):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    ks = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
          and "Memcpy" not in e.name and "Memset" not in e.name]
    ks.sort(key=lambda e: e.time_range.start)
    if not ks:
        print("no kernel records")
        return
    t0 = ks[0].time_range.start
    span = ks[-1].time_range.end - t0
    busy = sum(e.time_range.end - e.time_range.start for e in ks)
    gaps = []
    for a, b in zip(ks, ks[1:]):
        gaps.append(b.time_range.start - a.time_range.end)
    gaps_sorted = sorted(gaps)
    print(f"{cfg.name}: {len(ks)} kernels, span {span:.1f} us, busy {busy:.1f} us, "
          f"gaps {span - busy:.1f} us (median gap {gaps_sorted[len(gaps) // 2]:.2f} us)")
    agg = {}
    for e in ks:
        nm = e.name.replace("(anonymous namespace)::", "").split("(")[0].split("<")[0]
        nm = nm.replace("void ", "").split("::")[-1]
        d = e.time_range.end - e.time_range.start
        a = agg.setdefault(nm, [0, 0.0])
        a[0] += 1
        a[1] += d
    for nm, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {nm:36s} {n:4d} {t:9.1f} us  {100 * t / span:5.1f}%")


if __name__ == "__main__":
    main()
