#!/bin/bash
# Default work-item size per phase (capi_exec.cpp refine_chunk): parity + A/B against fixed 256 KiB items.
OUT=${OUT:-gpurun_out}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/${P:-s3}_pytest_gpu.log 2>&1; echo rc=$? >> $OUT/${P:-s3}_pytest_gpu.log
timeout 300 python tools/launch_latency.py > $OUT/${P:-s3}_launch_latency.json 2> $OUT/${P:-s3}_launch_latency.err
: > $OUT/${P:-s3}_small.jsonl
for w in tiny_tp2_to_dp2 data_gen_dp8_to_train_tp8 data_gen_dp8_to_pp2dp2tp2 llama7b_tp8_dp8_roundtrip; do
  for ck in 0 256; do
    timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --no-cpu --chunk-kib $ck 2>/dev/null | tail -1 >> $OUT/${P:-s3}_small.jsonl
  done
done
N=$(nvidia-smi -L | wc -l)
if [ "$N" -ge 2 ]; then
  for w in tiny_tp2_to_dp2 data_gen_dp8_to_train_tp8 data_gen_dp8_to_pp2dp2tp2; do
  for ck in 0 256; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29530 + ck / 64)) \
      bench.py --gpus 2 --workload $w --steps 50 --warmup 5 --no-e2e --chunk-kib $ck 2>/dev/null | tail -1 >> $OUT/${P:-s3}_small.jsonl
  done
  done
fi
