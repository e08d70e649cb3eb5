#!/bin/bash
# Kernel variant sweep on the flag-synchronised 7B round trip (overlap on) and the relay replicate.
N=$(nvidia-smi -L | wc -l)
make -s -C paper_2406_14088_b200/csrc >/dev/null
for w in "llama7b_tp8_dp8_roundtrip --overlap on" "llama7b_replicate_to_dp8 --mode relay"; do
  for k in 1 5 0; do  # 12, 13 pruned after round 1 (profiles/r01_flag_kernel_sweep_n{2,4}.txt)
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29516 bench.py --gpus $N --workload $w --kernel $k --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/q.log 2>&1
    echo "n=$N $w kernel=$k rc=$? $(tail -1 gpurun_out/q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["verified"])' 2>&1 | tail -1)"
  done
done | tee gpurun_out/flag_kernel_sweep_n$N.txt
