#!/bin/bash
# ncu evidence for the dominant kernel (run on the GPU box via gpurun, 1 GPU).
#   1. launch list (gpu__time_duration per launch) of the default bench command
#   2. one --set full capture of rr_copy_kernel (forward + back phase of one
#      step) on the same workload truncated to 2 decoder layers: ncu's kernel
#      replay saves/restores the written memory, which the full 144 GB
#      instance does not leave room for. Same kernel, same rectangle shapes.
# Each command first runs plainly (must exit 0) before it runs under ncu.
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
LIST_CMD="python bench.py --steps 3 --warmup 3 --cpu-budget 2 --e2e-steps 1"
FULL_CMD="python bench.py --steps 3 --warmup 3 --layers 2 --no-e2e --no-cpu"
$LIST_CMD > "$OUT/plain_list.log" 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$OUT/launches.csv" \
      $LIST_CMD > "$OUT/ncu_list.log" 2>&1
echo "launch list rc=$?"
$FULL_CMD > "$OUT/plain_full.log" 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:rr_copy_kernel -s 2 -c 2 \
      -o "$OUT/prof_copy" $FULL_CMD > "$OUT/ncu_full.log" 2>&1
echo "full capture rc=$?"
