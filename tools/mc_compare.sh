#!/bin/bash
# Multi-GPU: parity tests, then peer-store (push) vs NVLS multicast (mc) on
# the one-to-many workloads. Output: gpurun_out/mc_compare_n$N.txt
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_multigpu.py -x -q > "$OUT/pytest_mgpu_n$N.log" 2>&1
echo "pytest rc=$?"; tail -3 "$OUT/pytest_mgpu_n$N.log"
for w in llama7b_replicate_to_dp8 llama7b_tp8_dp8_roundtrip; do
  for m in push mc; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29513 bench.py --gpus $N --workload $w --mode $m --steps 10 --warmup 3 --no-e2e \
      > "$OUT/mc_${w}_${m}_n$N.log" 2>&1
    echo "$w $m rc=$? $(tail -1 "$OUT/mc_${w}_${m}_n$N.log" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["roofline"]["achieved"], d["verified"])' 2>&1 | tail -1)"
  done
done | tee "$OUT/mc_compare_n$N.txt"
for w in llama7b_replicate_to_dp8 llama7b_tp8_dp8_roundtrip; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29514 tools/nccl_compare.py --workload $w > "$OUT/nccl_${w}_n$N.log" 2>&1
  echo "$w nccl rc=$? $(tail -1 "$OUT/nccl_${w}_n$N.log")"
done | tee -a "$OUT/mc_compare_n$N.txt"
for w in llama7b_replicate_to_dp8; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29515 bench.py --gpus $N --workload $w --mode auto --steps 10 --warmup 3 --no-e2e \
    > "$OUT/auto_${w}_n$N.log" 2>&1
  echo "$w auto rc=$? $(tail -1 "$OUT/auto_${w}_n$N.log" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["config"]["multicast_sets"], d["verified"])' 2>&1 | tail -1)"
done | tee -a "$OUT/mc_compare_n$N.txt"
