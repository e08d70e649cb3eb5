#!/bin/bash
# Multi-GPU parity, then overlapped in-host fan-out on/off on the default workload and configs.
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_multigpu.py -x -q > "$OUT/pytest_mgpu_n$N.log" 2>&1
echo "pytest rc=$?"; tail -3 "$OUT/pytest_mgpu_n$N.log"
for w in llama7b_tp8_dp8_roundtrip llama13b_pp2tp4_to_dp2tp4 llama7b_replicate_to_dp8; do
  for o in off on; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29519 bench.py --gpus $N --workload $w --overlap $o --steps 10 --warmup 3 --no-e2e \
      > "$OUT/ov_${w}_${o}_n$N.log" 2>&1
    echo "$w overlap=$o rc=$? $(tail -1 "$OUT/ov_${w}_${o}_n$N.log" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["roofline"]["achieved"], d["config"]["relay_phases"], d["config"]["overlap_phases"], d["verified"])' 2>&1 | tail -1)"
  done
done | tee "$OUT/overlap_compare_n$N.txt"
