#!/bin/bash
# Multi-GPU parity (incl. relay) and push / relay / mc / nccl on the DP fan-out workloads.
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_multigpu.py -x -q > "$OUT/pytest_mgpu_n$N.log" 2>&1
echo "pytest rc=$?"; tail -3 "$OUT/pytest_mgpu_n$N.log"
for w in llama7b_replicate_to_dp8 llama7b_tp8_dp8_roundtrip; do
  for m in push relay mc auto; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29518 bench.py --gpus $N --workload $w --mode $m --steps 10 --warmup 3 --no-e2e \
      > "$OUT/rl_${w}_${m}_n$N.log" 2>&1
    echo "$w $m rc=$? $(tail -1 "$OUT/rl_${w}_${m}_n$N.log" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["roofline"]["achieved"], d["config"]["relay_phases"], d["verified"])' 2>&1 | tail -1)"
  done
done | tee "$OUT/relay_compare_n$N.txt"
