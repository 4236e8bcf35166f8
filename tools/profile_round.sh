#!/usr/bin/env bash
# ncu evidence for profiles/ (run on the GPU box from the repo root, one GPU):
#   1. launch lists (gpu__time_duration per launch) of the TIMED steps of the
#      bench command (NVTX range lr_timed) for cfg2 (default) and cfg4;
#   2. one `--set full` capture of each hot kernel: the first two passes over
#      A (NVTX range lr_pass: A.Omega and A^T.Q), the Cholesky and Jacobi
#      kernels of the timed steps.
# Each bench command first runs once without ncu (it must exit 0).
set -u
OUT=${OUT:-gpurun_out/prof}
CONFIGS=${CONFIGS:-"2 4 5"}
mkdir -p "$OUT"
NCU=/usr/local/cuda/bin/ncu
for C in $CONFIGS; do
  B="python bench.py --config $C --steps 2 --warmup 3 --no-e2e --no-cpu"
  $B > "$OUT/bench_cfg$C.json" 2> "$OUT/bench_cfg$C.err" || { echo "bench cfg$C failed"; continue; }
  [ -n "${SKIP_LAUNCHES:-}" ] || $NCU --nvtx --nvtx-include "lr_timed/" --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file "$OUT/launches_cfg$C.csv" $B > /dev/null 2>&1
  # the pass kernels by name (the timed steps replay a CUDA graph, whose
  # nodes carry no NVTX ranges): skip the warm-up launches, capture two
  $NCU --set full --clock-control none --import-source on \
    -k regex:"${PASS_KERNELS:-gemm_f64_tma_kernel|gemm_f32_tc_kernel|csr_spmm}" -s ${PASS_SKIP:-6} -c ${PASS_COUNT:-2} \
    -o "$OUT/full_cfg${C}_pass" -f $B > /dev/null 2>&1
  [ -n "${SKIP_SMALL:-}" ] || $NCU --nvtx --nvtx-include "lr_timed/" --set full --clock-control none --import-source on \
    -k regex:"${SMALL_KERNELS:-chol|jacobi}" -c 2 -o "$OUT/full_cfg${C}_small" -f $B > /dev/null 2>&1
done
ls -la "$OUT"
