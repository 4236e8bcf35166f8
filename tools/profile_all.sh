#!/usr/bin/env bash
# Round evidence for every BASELINE config (run on the GPU box, repo root):
# per-config pass-kernel regex for the --set full capture.
set -u
OUT=${OUT:-gpurun_out/prof}
run() { OUT=$OUT CONFIGS="$1" PASS_KERNELS="$2" PASS_SKIP=${3:-6} bash tools/profile_round.sh; }
run 2 "ozaki_gemm"
run 1 "gemm_f64_kernel" 12
run 3 "gemm_f32_tc_kernel"
run 4 "gemm_f32_tc_kernel"
run 5 "csr_spmm"
ls -la "$OUT"
