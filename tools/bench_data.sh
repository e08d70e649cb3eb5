#!/bin/bash
# Data-transfer workloads (plan_data_transfer) at 1 GPU and
# at every GPU of the box: one bench JSON line per (workload, N).
N=$(nvidia-smi -L | wc -l)
OUT=${OUT:-gpurun_out/bench_data.jsonl}
: > $OUT
for wl in data_gen_dp8_to_train_tp8 data_gen_dp8_to_pp2dp2tp2; do
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 >> $OUT
  if [ "$N" -gt 1 ]; then
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29531 bench.py --gpus $N --workload $wl --steps 20 --warmup 5 2>/dev/null | tail -1 >> $OUT
  fi
done
