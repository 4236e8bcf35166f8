#!/usr/bin/env bash
# ncu launch lists (gpu__time_duration per launch) of the timed steps of
# bench.py for the given configs; each bench command first runs without ncu.
set -u
OUT=${OUT:-gpurun_out/ll}
CONFIGS=${CONFIGS:-"1 2 3 4 5"}
mkdir -p "$OUT"
NCU=/usr/local/cuda/bin/ncu
for C in $CONFIGS; do
  B="python bench.py --config $C --steps 1 --warmup 3 --no-e2e --no-cpu"
  $B > "$OUT/bench_cfg$C.json" 2> "$OUT/bench_cfg$C.err" || { echo "bench cfg$C failed"; continue; }
  $NCU --nvtx --nvtx-include "lr_timed/" --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file "$OUT/launches_cfg$C.csv" $B > /dev/null 2>&1
done
ls -la "$OUT"
