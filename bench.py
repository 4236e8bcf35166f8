"""Benchmark: rank-k randomized SVD on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One step = one rank-k randomized SVD of the configuration's A as the
reference CLI composes it (cli.py:128-165 Stage A + direct_svd; SURVEY.md
§8a a13): Stage A (Alg 4.1 / 4.4 / 4.5) + Alg 5.1, i.e. 2q+2 passes over A.
The posterior estimator (one more pass, r = 10) is timed separately, as in
the reference's CPU plan.

value = whole-job A-GB/s = passes x bytes(A) / step time (higher is better);
ms_per_step is the rSVD time.  A is device-resident before timing starts;
A (>= 1 GiB for the default config) exceeds the 126 MB L2, so no explicit
flush is needed between steps.  `e2e` repeats the measurement through the
public API with host buffers: the pinned host A is copied to the device,
validated, factored, and U / sigma / V copied back, every step.

--impl reference times the CPU oracle (oracle/lowrank_oracle.py, a numpy
restatement of the reference package, pinned to the reference's golden
vectors) on the host cores with all BLAS threads.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=4,
                   help="BASELINE.json config (default 4: the largest single-GPU config, "
                        "north_star's row-sharded scaling config)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--sharded", action="store_true",
                   help="use the row-sharded (NCCL) path even at one GPU")
    return p.parse_args()


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.th = None

    def _run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# inputs

def build_input(cfg, device="cuda"):
    """Device-resident A for the configuration (see workloads.py)."""
    import torch
    if cfg.idx in (1, 2):
        A, _ = workloads.build_synthetic_device(cfg.m, cfg.n, workloads.spectrum(cfg.idx, cfg.n),
                                                cfg.seed, device=device)
        return A
    if cfg.idx == 3:
        return torch.from_numpy(workloads.build_cfg3()).to(device)
    if cfg.idx == 4:
        A, _ = workloads.build_cfg4_device(device=device)
        return A
    raise ValueError("config 5 is built by build_sparse")


def measured_fp64_peak():
    """cuBLAS DGEMM 8192^3 (best of 5) -- the FP64 tensor peak the roofline
    uses (MEASURED_PEAKS.json has only HBM and bf16)."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    del a, b
    return 2.0 * n ** 3 / best / 1e12


def measured_int8_peak():
    """cuBLASLt int8 GEMM 8192^3 (torch._int_mm, best of 5) in TOP/s -- the
    int8 tensor peak of the emulated fp64 passes (not in MEASURED_PEAKS.json)."""
    import torch
    n = 8192
    a = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda")
    for _ in range(2):
        torch._int_mm(a, b)
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch._int_mm(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    del a, b
    return 2.0 * n ** 3 / best / 1e12


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def config_dict(cfg, world):
    """The `config` object of every line (both arms, every N): identical
    keys and values so the driver can match them."""
    return {"workload": cfg.name, "config_index": cfg.idx, "m": cfg.m, "n": cfg.n,
            "k": cfg.k, "ell": cfg.ell, "q": cfg.q, "sketch": cfg.sketch,
            "passes": cfg.passes(), "a_bytes": cfg.a_bytes(),
            "a_bytes_model": ("CSR values f64 + int32 cols + int64 rowptr" if cfg.idx == 5
                              else "dense A in its storage dtype"),
            "l2": "inputs larger than the 126 MB L2 (A >= 512 MiB per GPU), no flush",
            "parallelism": f"row-sharded x{world}" if world > 1 else "single GPU"}


def cpu_baseline(cfg, A_dev=None):
    """The CPU oracle (kind "port": numpy/OpenBLAS with all host threads) on
    a bounded sample of the same workload; returns the line's cpu_baseline
    object (rate in A-GB/s = passes x sample bytes / seconds)."""
    from oracle import lowrank_oracle as O
    op, a_bytes, sample = reference_sample(cfg, A_dev)
    t0 = time.perf_counter()
    O.rsvd(op, cfg.k, cfg.p, cfg.q, cfg.seed, sketch=cfg.sketch, estimate=False)
    dt = time.perf_counter() - t0
    return {"value": round(cfg.passes() * a_bytes / dt / 1e9, 4), "unit": "A-GB/s",
            "cores": os.cpu_count(), "kind": "port",
            "sample": f"{sample}: one rSVD (Stage A + direct SVD) by oracle/lowrank_oracle.py, "
                      f"{dt:.2f} s", "seconds": round(dt, 3)}


# ---------------------------------------------------------------------------

def run_ours(args, cfg):
    import torch
    import paper_0909_4061_b200 as lr
    from paper_0909_4061_b200 import core as lrcore

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1 or args.sharded:
        return run_sharded(args, cfg)
    if cfg.idx == 5:
        return run_sparse(args, cfg)
    A = build_input(cfg)
    torch.cuda.synchronize()
    op = lr.DenseOperator(A)
    a_bytes = A.numel() * A.element_size()
    passes = cfg.passes()

    def step():
        return lr.randomized_svd(op, cfg.k, cfg.p, cfg.q, cfg.seed, sketch=cfg.sketch,
                                 estimate=False)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # timed region: K steps, CUDA events on the launching stream
    lrcore.PASS_EVENTS = []
    l0 = lr._lib.launch_count()
    with ClockSampler(local) as clk:
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.nvtx.range_push("lr_timed")  # ncu --nvtx-include lr_timed/
        s.record()
        for _ in range(args.steps):
            step()
        e.record()
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
    launches = lr._lib.launch_count() - l0
    ms = s.elapsed_time(e) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    pev = lrcore.PASS_EVENTS
    lrcore.PASS_EVENTS = None

    # estimator pass, timed separately
    est_s, est_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b, f, _ = step()
    lr.posterior_error_estimate(op, b.Q, r=10, alpha=10.0, seed=cfg.seed + 13)   # warm-up
    torch.cuda.synchronize()
    est_s.record()
    est = lr.posterior_error_estimate(op, b.Q, r=10, alpha=10.0, seed=cfg.seed + 13)
    est_e.record()
    torch.cuda.synchronize()
    est_ms = est_s.elapsed_time(est_e)

    value = passes * a_bytes / (ms / 1e3) / 1e9
    roof = roofline(A, cfg, pev, ms, args.steps, passes, a_bytes)
    line = {
        "metric": "rank-k rSVD time & A-GB/s (% roofline) at 1/2/4/8 B200 vs host-CPU ref",
        "value": round(value, 3), "unit": "A-GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": {torch.float64: "f64", torch.float32: "f32", torch.complex64: "c64",
                  torch.complex128: "c128"}[A.dtype],
        "data": "synthetic (seeded, BASELINE.json config recipe; see workloads.py)",
        "config": config_dict(cfg, world),
        "roofline": roof,
        "estimator_ms": round(est_ms, 4),
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }

    if not args.no_e2e and rank == 0:
        line["e2e"] = e2e_measure(args, cfg, A, lr)
    if A.dtype == torch.float64 and lrcore._ozaki_wanted(
            A, torch.empty((1, cfg.ell), dtype=A.dtype, device=A.device)):
        # the int8 digit planes are built once per operator (cached on A) and
        # are not part of the timed steps: their build time, reported here
        ps, pe = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ps.record()
        lrcore.ozaki_prepare(A)
        pe.record()
        torch.cuda.synchronize()
        line["digit_plane_build_ms"] = round(ps.elapsed_time(pe), 4)
        line["digit_plane_build_note"] = (
            "once per operator (reads A, writes 2 x A's bytes); outside the timed steps, "
            "inside every e2e step")
    if not args.no_cpu and rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baseline(cfg, A)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def roofline_sparse(cfg, pev, ms, steps, passes):
    """Config 5: the dominant kernel is the CSR SpMM (K6), HBM bound;
    achieved = compulsory bytes per launch (CSR arrays, X once, Y) / launch
    time."""
    pk, src = peaks()
    t = [a.elapsed_time(b) for a, b, *_ in pev]
    nbytes = [x for _, _, _, x, _ in pev]
    avg_ms = sum(t) / len(t)
    achieved = sum(nbytes) / len(nbytes) / (avg_ms / 1e3) / 1e9
    hbm = pk["hbm_gbs"]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(f"cfg{cfg.idx}")
    # cache-capacity-aware bound for UNIFORMLY RANDOM column indices: a gathered
    # row of X (8 ell bytes) is in L2 only if it was touched recently; with the
    # n x ell panel far larger than the cache (805 MB against 126 MB at config 5)
    # the expected hit rate is ~ L2 / |X|, whatever the schedule -- the
    # compulsory model (X read once) is not attainable for this matrix
    ell = pev[0][4]
    l2 = 126e6
    x_bytes = cfg.n * ell * 8
    miss = max(0.0, 1.0 - l2 / x_bytes)
    nnz = pev[0][2] / (2.0 * ell)          # the launch's flops are 2 nnz ell
    cap_bound = sum(nbytes) / len(nbytes) + miss * max(nnz - cfg.n, 0) * ell * 8
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(achieved / hbm, 4), "traffic": traffic,
            "capacity_bound_bytes": int(cap_bound),
            "traffic_over_capacity_bound": round(traffic / cap_bound, 3) if traffic else None,
            "kernel": "csr_spmm (K6: half-warp gathers), compulsory bytes model; "
                      "capacity_bound_bytes = expected DRAM bytes with random columns and a 126 MB L2",
            "peak_source": f"{src} HBM copy bandwidth (MEASURED_PEAKS.json)",
            "avg_spmm_ms": round(avg_ms, 4),
            "dram_frac_measured_traffic": (round(traffic / (avg_ms / 1e3) / 1e9 / hbm, 4)
                                           if traffic else None),
            "spmm_share_of_step": round(sum(t) / (ms * steps), 4)}


def roofline(A, cfg, pev, ms, steps, passes, a_bytes):
    """Roofline of the dominant kernel (the pass over A, K1/K2), from the
    CUDA events recorded around every pass inside the timed region."""
    import torch
    pass_ms = [a.elapsed_time(b) for a, b, *_ in pev]
    flops_per = [f for _, _, f, _, _ in pev]
    avg_pass_ms = sum(pass_ms) / len(pass_ms)
    avg_flops = sum(flops_per) / len(flops_per)
    pk, src = peaks()
    from paper_0909_4061_b200 import core as lrcore
    ozaki = A.dtype == torch.float64 and lrcore._ozaki_wanted(
        A, torch.empty((1, cfg.ell), dtype=A.dtype, device=A.device))
    if A.dtype in (torch.float64, torch.complex128):
        peak_tf = measured_fp64_peak()
        peak_src = "measured in-run: cuBLAS DGEMM 8192^3 (torch.matmul)"
    else:
        # burst figure for a pass in a short step, the sustained one for a
        # pass inside a long step (config 4: 4 x 5.5 ms of back-to-back
        # tensor work per step; the clocks drop to ~1.3 GHz under that load,
        # profiles/round2_m256_pass_summary.md)
        long_step = ms >= 10.0 and "bf16_tflops_sustained" in pk
        peak_tf = pk["bf16_tflops_sustained"] if long_step else pk["bf16_tflops"]
        peak_src = (f"{src} bf16 {'sustained' if long_step else 'burst'} (MEASURED_PEAKS.json)")
    achieved_tf = avg_flops / (avg_pass_ms / 1e3) / 1e12
    hbm = pk["hbm_gbs"]
    # per-pass roofline: max(flops / tensor peak, bytes(A) / HBM)
    roof_pass_s = max(avg_flops / (peak_tf * 1e12), a_bytes / (hbm * 1e9))
    roof_step_ms = passes * roof_pass_s * 1e3
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(f"cfg{cfg.idx}")
    if ozaki:
        # fp64 passes emulated on the int8 tensor cores (lr_gemm_ozaki): the
        # kernel's own bound is int8 work -- 36 digit-plane products over
        # 64-column tiles -- against the measured int8 peak; the fp64-DMMA
        # roofline (the native fp64 bound) is kept beside it
        i8_peak = measured_int8_peak()
        m, n = A.shape
        # the tensor work the kernel issues (gemm_f64_ozaki.cu): CTA pairs
        # (>= 8192 output rows, 56-column tiles) 20 UMMAs of 2 x 56 columns per
        # 32-deep stage = 40 digit products per tile column; single CTAs 36
        # products over 64-column tiles (32 when l <= 32)
        # algorithmic int8 work only: the 36 digit products (s + t <= 9) over
        # the ell real columns -- not the padded tile columns nor the extra
        # 10th-diagonal products the CTA-pair kernel issues
        i8_ops = 36 * 2.0 * m * n * cfg.ell
        achieved_i8 = i8_ops / (avg_pass_ms / 1e3) / 1e12
        roof_i8_s = max(i8_ops / (i8_peak * 1e12), a_bytes / (hbm * 1e9))
        return {"bound": "tensor", "achieved": round(achieved_i8, 1), "peak": round(i8_peak, 1),
                "unit": "TOP/s (int8)", "frac": round(achieved_i8 / i8_peak, 4),
                "traffic": traffic,
                "kernel": "ozaki_gemm2_kernel (CTA pairs; ozaki_gemm_kernel below 8192 "
                          "output rows): fp64 pass over A as 36 exact int8 digit-plane "
                          "products on tcgen05 (lr_gemm_ozaki)",
                "peak_source": "measured in-run: cuBLASLt int8 GEMM 8192^3 (torch._int_mm)",
                "int8_ops_per_pass": i8_ops,
                "avg_pass_ms": round(avg_pass_ms, 4),
                "fp64_equiv_tflops": round(achieved_tf, 3),
                "fp64_dmma_peak_tflops": round(peak_tf, 3),
                "fp64_equiv_frac_of_dmma_peak": round(achieved_tf / peak_tf, 4),
                "pass_a_gbs": round(a_bytes / (avg_pass_ms / 1e3) / 1e9, 1),
                "hbm_frac": round(a_bytes / (avg_pass_ms / 1e3) / 1e9 / hbm, 4),
                "step_roofline_ms": round(roof_step_ms, 4),
                "step_roofline_frac": round(roof_step_ms / ms, 4),
                "step_roofline_basis": "fp64 flops at the DMMA peak vs A bytes at HBM, per pass",
                "step_roofline_int8_ms": round(passes * roof_i8_s * 1e3, 4),
                "step_roofline_int8_frac": round(passes * roof_i8_s * 1e3 / ms, 4),
                "pass_share_of_step": round(sum(pass_ms) / (ms * steps), 4)}
    if A.dtype in (torch.float32, torch.complex64):
        # the tcgen05 pass issues three fp16 products per algorithmic product
        # (hi*hi + hi*lo + lo*hi): the kernel's own
        # bound is that tensor work at the bf16/fp16 peak; the north_star step
        # roofline (per pass max(2mnl at the 1x-TF32 rate, A bytes at HBM)) is
        # HBM-bound for fp32 and is reported beside it
        issued = 3.0 * avg_flops
        ach3 = issued / (avg_pass_ms / 1e3) / 1e12
        roof_pass_s = max(avg_flops / (0.5 * peak_tf * 1e12), a_bytes / (hbm * 1e9))
        roof_step_ms = passes * roof_pass_s * 1e3
        return {"bound": "tensor", "achieved": round(ach3, 3), "peak": round(peak_tf, 3),
                "unit": "TFLOP/s (fp16 issued)", "frac": round(ach3 / peak_tf, 4),
                "traffic": traffic,
                "kernel": "gemm_f32_tc pass over A (tcgen05 kind::f16, 3-product split)",
                "peak_source": peak_src, "avg_pass_ms": round(avg_pass_ms, 4),
                "algorithmic_tflops": round(achieved_tf, 3),
                "issued_flops_per_pass": issued,
                "frac_of_burst_peak": round(ach3 / pk["bf16_tflops"], 4),
                "pass_a_gbs": round(a_bytes / (avg_pass_ms / 1e3) / 1e9, 1),
                "hbm_frac": round(a_bytes / (avg_pass_ms / 1e3) / 1e9 / hbm, 4),
                "step_roofline_ms": round(roof_step_ms, 4),
                "step_roofline_frac": round(roof_step_ms / ms, 4),
                "step_roofline_basis": "per pass max(2mnl at 1x TF32 = half the bf16 peak, "
                                       "A bytes at HBM) -- HBM-bound",
                "step_roofline_3product_ms": round(passes * max(
                    issued / (peak_tf * 1e12), a_bytes / (hbm * 1e9)) * 1e3, 4),
                "pass_share_of_step": round(sum(pass_ms) / (ms * steps), 4)}
    return {"bound": "tensor", "achieved": round(achieved_tf, 3), "peak": round(peak_tf, 3),
            "unit": "TFLOP/s", "frac": round(achieved_tf / peak_tf, 4),
            "traffic": traffic, "kernel": "lr_gemm pass over A (K1/K2)",
            "peak_source": peak_src, "avg_pass_ms": round(avg_pass_ms, 4),
            "pass_a_gbs": round(a_bytes / (avg_pass_ms / 1e3) / 1e9, 1),
            "hbm_frac": round(a_bytes / (avg_pass_ms / 1e3) / 1e9 / hbm, 4),
            "step_roofline_ms": round(roof_step_ms, 4),
            "step_roofline_frac": round(roof_step_ms / ms, 4),
            "pass_share_of_step": round(sum(pass_ms) / (ms * steps), 4)}


def run_sparse(args, cfg):
    """Config 5: CSR S (2^21 x 2^21, ~16 nnz/row) + implicit L R^T, q = 3."""
    import torch
    import paper_0909_4061_b200 as lr
    from paper_0909_4061_b200 import core as lrcore
    rank, world, local = env_rank()
    S, L, R = workloads.build_cfg5()
    op = lr.CudaCsrOperator(S, L, R)
    a_bytes = op.csr_bytes()
    passes = cfg.passes()

    def step():
        return lr.randomized_svd(op, cfg.k, cfg.p, cfg.q, cfg.seed, estimate=False)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    lrcore.PASS_EVENTS = []
    l0 = lr._lib.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.nvtx.range_push("lr_timed")
        s.record()
        for _ in range(args.steps):
            step()
        e.record()
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
    launches = lr._lib.launch_count() - l0
    ms = s.elapsed_time(e) / args.steps
    pev = lrcore.PASS_EVENTS
    lrcore.PASS_EVENTS = None
    line = {
        "metric": "rank-k rSVD time & A-GB/s (% roofline) at 1/2/4/8 B200 vs host-CPU ref",
        "value": round(passes * a_bytes / (ms / 1e3) / 1e9, 3), "unit": "A-GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded CSR + Gaussian low-rank factors, BASELINE.json config 5)",
        "config": config_dict(cfg, world),
        "roofline": roofline_sparse(cfg, pev, ms, args.steps, passes),
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if not args.no_e2e and rank == 0:
        # end to end: scipy CSR + numpy factors on the host in (operator built
        # per call: upload, device-side transpose), numpy factors out
        def once():
            o = lr.CudaCsrOperator(S, L, R, host_io=True)
            return lr.randomized_svd(o, cfg.k, cfg.p, cfg.q, cfg.seed, estimate=False)
        for _ in range(3):
            res = once()
        torch.cuda.synchronize()
        k_e2e = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            res = once()
        dt = (time.perf_counter() - t0) / k_e2e
        f = res[1]
        h2d = S.data.nbytes + S.indices.nbytes + (S.shape[0] + 1) * 8 + L.nbytes + R.nbytes
        d2h = res[0].Q.nbytes + f.U.nbytes + f.sigma.nbytes + f.V.nbytes
        line["e2e"] = {"value": round(passes * a_bytes / dt / 1e9, 3), "unit": "A-GB/s",
                       "ms_per_step": round(dt * 1e3, 3), "h2d_bytes_per_step": int(h2d),
                       "d2h_bytes_per_step": int(d2h), "steps": k_e2e}
    if not args.no_cpu and rank == 0:
        line["cpu_baseline"] = cpu_baseline(cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)



def run_sharded(args, cfg):
    """N GPUs, A split by rows (paper_0909_4061_b200.dist): Omega replicated,
    Gram and n x ell partials all-reduced over NCCL.  Strong scaling: the
    whole A is fixed, each rank holds m/N rows."""
    import torch
    import torch.distributed as dist
    import paper_0909_4061_b200 as lr
    from paper_0909_4061_b200 import core as lrcore
    from paper_0909_4061_b200.dist import (Comm, GpuBackend, dist_randomized_svd, row_range,
                                           sharded_randomized_svd)
    rank, world, local = env_rank()
    os.environ.setdefault("NCCL_DEBUG", "INFO")     # rank/NVLink setup in the log
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29533", rank=0,
                                world_size=1, device_id=torch.device("cuda", local))
    if cfg.idx == 5:
        return run_sharded_sparse(args, cfg, rank, world, local)
    if cfg.idx == 4:
        # each rank builds only its rows (the recipe is blockwise)
        r0, r1 = row_range(cfg.m, rank, world)
        A, _ = workloads.build_cfg4_device(rows=(r0, r1))
        m_total, n = cfg.m, cfg.n
        a_bytes_total = cfg.a_bytes()
    else:
        A_full = build_input(cfg)
        r0, r1 = row_range(A_full.shape[0], rank, world)
        A = A_full[r0:r1].contiguous()
        m_total, n = A_full.shape
        a_bytes_total = A_full.numel() * A_full.element_size()
        del A_full
    torch.cuda.empty_cache()
    comm, be = Comm(), GpuBackend()
    op = lr.DenseOperator(A)
    amax = None
    if A.dtype in (torch.float32, torch.complex64):
        t = torch.tensor([op.amax], dtype=torch.float64, device="cuda")
        amax = float(comm.allreduce_max(t).item())
    passes = cfg.passes()
    sketch = "srft" if cfg.sketch == "srft" else "gauss"

    def step(estimate=False):
        return dist_randomized_svd(A, n, cfg.k, cfg.p, cfg.q, cfg.seed, comm, be, amax=amax,
                                   estimate=estimate, sketch=sketch)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    lrcore.PASS_EVENTS = []
    l0 = lr._lib.launch_count()
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.nvtx.range_push("lr_timed")  # ncu --nvtx-include lr_timed/
        s.record()
        for _ in range(args.steps):
            step()
        e.record()
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        dist.barrier()
    launches = lr._lib.launch_count() - l0
    ms_local = s.elapsed_time(e) / args.steps
    t = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    pev = lrcore.PASS_EVENTS
    lrcore.PASS_EVENTS = None
    a_bytes_local = A.numel() * A.element_size()
    roof = roofline(A, cfg, pev, ms_local, args.steps, passes, a_bytes_local)

    est_s, est_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    est_s.record()
    res = step(estimate=True)
    est_e.record()
    torch.cuda.synchronize()

    line = {
        "metric": "rank-k rSVD time & A-GB/s (% roofline) at 1/2/4/8 B200 vs host-CPU ref",
        "value": round(passes * a_bytes_total / (ms / 1e3) / 1e9, 3), "unit": "A-GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None,
        "dtype": {torch.float64: "f64", torch.float32: "f32", torch.complex64: "c64",
                  torch.complex128: "c128"}[A.dtype],
        "data": "synthetic (seeded, BASELINE.json config recipe; see workloads.py)",
        "config": config_dict(cfg, world),
        "rows_per_rank": r1 - r0,
        "roofline": roof,
        "rsvd_plus_estimate_ms_rank0": round(est_s.elapsed_time(est_e), 4),
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if not args.no_e2e:
        host = torch.empty(A.shape, dtype=A.dtype, pin_memory=True)
        host.copy_(A)
        A_np = host   # pinned CPU rows (async H2D)
        k_e2e = max(1, min(args.steps, 5))
        sharded_randomized_svd(A_np, cfg.k, cfg.p, cfg.q, cfg.seed, sketch=sketch,
                               estimate=False)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            U, S, V, _ = sharded_randomized_svd(A_np, cfg.k, cfg.p, cfg.q, cfg.seed,
                                                sketch=sketch, estimate=False)
        dt = (time.perf_counter() - t0) / k_e2e
        tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        line["e2e"] = {"value": round(passes * a_bytes_total / dt / 1e9, 3), "unit": "A-GB/s",
                       "ms_per_step": round(dt * 1e3, 3),
                       "h2d_bytes_per_step": int(a_bytes_total),
                       "d2h_bytes_per_step": int(U.nbytes * world + S.nbytes + V.nbytes),
                       "steps": k_e2e, "timing": "wall clock per rank, max over ranks"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()



def run_sharded_sparse(args, cfg, rank, world, local):
    """Config 5 on N GPUs: rank r holds rows row_range(2^21, r, N) of S and L
    (R replicated) as a CudaCsrOperator; the n-side panels are sharded too
    (all-gather before A_r X, reduce-scatter after A_r^H Y --
    dist_randomized_svd_operator).  Strong scaling."""
    import torch
    import torch.distributed as dist
    import paper_0909_4061_b200 as lr
    from paper_0909_4061_b200 import core as lrcore
    from paper_0909_4061_b200.dist import Comm, GpuBackend, dist_randomized_svd_operator, row_range
    S, L, R = workloads.build_cfg5()
    n = S.shape[0]
    a, b = row_range(n, rank, world)
    op = lr.CudaCsrOperator(S[a:b], L[a:b], R)
    nnz_total = int(S.nnz)
    del S
    comm, be = Comm(), GpuBackend()
    passes = cfg.passes()
    a_bytes = cfg.a_bytes(nnz_total)

    def step(estimate=False):
        return dist_randomized_svd_operator(op, n, cfg.k, cfg.p, cfg.q, cfg.seed, comm, be,
                                            estimate=estimate)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    lrcore.PASS_EVENTS = []
    l0 = lr._lib.launch_count()
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            step()
        e.record()
        torch.cuda.synchronize()
        dist.barrier()
    launches = lr._lib.launch_count() - l0
    t = torch.tensor([s.elapsed_time(e) / args.steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    pev = lrcore.PASS_EVENTS
    lrcore.PASS_EVENTS = None
    line = {
        "metric": "rank-k rSVD time & A-GB/s (% roofline) at 1/2/4/8 B200 vs host-CPU ref",
        "value": round(passes * a_bytes / (ms / 1e3) / 1e9, 3), "unit": "A-GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded CSR + Gaussian low-rank factors, BASELINE.json config 5)",
        "config": config_dict(cfg, world),
        "rows_per_rank": b - a,
        "roofline": roofline_sparse(cfg, pev, ms, args.steps, passes),
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def e2e_measure(args, cfg, A, lr):
    """Same metric through the public API with pinned host buffers."""
    import torch
    host = torch.empty(A.shape, dtype=A.dtype, pin_memory=True)
    host.copy_(A)
    steps = max(1, min(args.steps, 5))

    def once():
        # pinned CPU tensor in (async H2D at full PCIe rate), numpy factors out
        b, f, _ = lr.randomized_svd(host, cfg.k, cfg.p, cfg.q, cfg.seed, sketch=cfg.sketch,
                                    estimate=False)
        return b, f

    # warm-up: allocator / pinned-buffer caches settle by the 3rd call.  The
    # previous call's factors stay referenced while the next call runs, as in
    # the timed loop (their pinned host buffers are then not recycled: the
    # second set is allocated here, ~0.5 s of page pinning, not in a timed call)
    for _ in range(3):
        f = once()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    per_call = []
    for _ in range(steps):
        tc = time.perf_counter()
        b, f = once()
        per_call.append(time.perf_counter() - tc)
    dt = (time.perf_counter() - t0) / steps
    if os.environ.get("LR_E2E_DEBUG"):
        print("e2e per call (ms):", [round(1e3 * x, 1) for x in per_call], file=sys.stderr)
    a_bytes = A.numel() * A.element_size()
    d2h = b.Q.nbytes + f.U.nbytes + f.sigma.nbytes + f.V.nbytes   # the basis comes back too
    return {"value": round(cfg.passes() * a_bytes / dt / 1e9, 3), "unit": "A-GB/s",
            "ms_per_step": round(dt * 1e3, 3), "h2d_bytes_per_step": int(a_bytes),
            "d2h_bytes_per_step": int(d2h), "steps": steps}


def reference_sample(cfg, A_dev=None):
    """(operator, A-bytes of one pass, sample description) for the CPU legs
    (reference arm, cpu_baseline): the full matrix where one CPU rSVD takes
    seconds (configs 1, 2), otherwise a bounded sample of the same recipe --
    rows of the same matrix, so the A-GB/s rate is comparable."""
    from oracle import lowrank_oracle as O
    import torch
    if cfg.idx in (1, 2):
        if A_dev is not None:
            A = A_dev.cpu().numpy()
        elif torch.cuda.is_available():
            A = build_input(cfg).cpu().numpy()
            torch.cuda.empty_cache()
        else:
            A, _ = workloads.synthetic_explicit(cfg.m, cfg.n, workloads.spectrum(cfg.idx, cfg.n),
                                                cfg.seed)
        return O.Dense(A), A.size * A.itemsize, f"full {cfg.name} matrix"
    if cfg.idx == 3:
        A = A_dev[:1024].cpu().numpy() if A_dev is not None else workloads.build_cfg3()[:1024]
        return O.Dense(A), A.size * A.itemsize, "config-3 matrix, first 1024 of 8192 rows"
    if cfg.idx == 4:
        rows = 65536
        A = (A_dev[:rows].cpu().numpy() if A_dev is not None
             else workloads.cfg4_block_host(0))
        return (O.Blockwise(A), A.size * 4,
                f"config-4 matrix, first {rows} of 2^20 rows (recipe block 0), fp64 "
                "row-block application (O.Blockwise)")
    S, L, R = workloads.build_cfg5(n=1 << 17)
    return (O.SparsePlusLowRank(S, L, R), S.nnz * 12 + (S.shape[0] + 1) * 8,
            "config-5 recipe at n = 2^17 (scipy CSR, single-threaded SpMM)")


def run_reference(args, cfg):
    """--impl reference: the reference algorithm's CPU implementation (the
    oracle port of the pure-Python reference package, numpy/OpenBLAS with
    all host threads) on the same recipe; rank 0 only under torchrun."""
    rank, world, local = env_rank()
    if rank != 0:
        return
    import torch
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    from oracle import lowrank_oracle as O
    op, a_bytes, sample = reference_sample(cfg)
    for _ in range(args.warmup):
        O.rsvd(op, cfg.k, cfg.p, cfg.q, cfg.seed, sketch=cfg.sketch, estimate=False)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.rsvd(op, cfg.k, cfg.p, cfg.q, cfg.seed, sketch=cfg.sketch, estimate=False)
    dt = (time.perf_counter() - t0) / args.steps
    v = cfg.passes() * a_bytes / dt / 1e9
    line = {
        "metric": "rank-k rSVD time & A-GB/s (% roofline) at 1/2/4/8 B200 vs host-CPU ref",
        "impl": "reference", "value": round(v, 4), "unit": "A-GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": {"f64": "f64", "f32": "f64 (reference upcast)", "c64": "c128 (reference upcast)"
                  }.get(cfg.dtype, "f64"),
        "data": "synthetic (seeded, BASELINE.json config recipe; see workloads.py)",
        "config": config_dict(cfg, world),
        "cpu_baseline": {"value": round(v, 4), "unit": "A-GB/s", "cores": os.cpu_count(),
                         "kind": "port",
                         "sample": f"{sample}: one rSVD (Stage A + direct SVD) per step by "
                                   "oracle/lowrank_oracle.py, numpy/OpenBLAS, all host threads"},
        "e2e": {"value": round(v, 4), "unit": "A-GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args):
    """bench.py --gpus N run directly (not under torchrun): re-launch this
    script as N ranks, one per GPU, with torch.distributed.run on 127.0.0.1
    (NCCL_DEBUG=INFO so every rank's NCCL init is visible in the log)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn_ranks(args))
    cfg = workloads.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
