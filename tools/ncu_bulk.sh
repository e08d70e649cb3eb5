#!/bin/bash
# ncu evidence for the default copy engine (rr_bulk_kernel), 1 GPU:
#  1. launch list of the default bench command;
#  2. DRAM bytes + duration of the full-size forward launch (single-pass
#     metrics: no kernel replay, so no save/restore of the 144 GB working set);
#  3. --set full capture (forward + back) on the 2-layer instance for stalls.
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
LIST_CMD="python bench.py --steps 3 --warmup 3 --cpu-budget 2 --e2e-steps 1"
$LIST_CMD > "$OUT/plain_list.log" 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$OUT/launches_bulk.csv" \
      $LIST_CMD > "$OUT/ncu_list.log" 2>&1
echo "launch list rc=$?"
FULL="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$FULL > "$OUT/plain_fullsize.log" 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
      --clock-control none -k regex:rr_bulk_kernel -s 6 -c 2 --csv --log-file "$OUT/dram_fullsize.csv" \
      $FULL > "$OUT/ncu_fullsize.log" 2>&1
echo "full-size dram rc=$?"
SMALL="python bench.py --steps 3 --warmup 3 --layers 2 --no-e2e --no-cpu"
$SMALL > "$OUT/plain_small.log" 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:rr_bulk_kernel -s 6 -c 2 \
      -o "$OUT/prof_bulk" $SMALL > "$OUT/ncu_small.log" 2>&1
echo "full capture rc=$?"
