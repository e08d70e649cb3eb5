#!/bin/bash
# Flag-synchronised phases (overlap / relay) on the TMA bulk kernel vs the LDG/STG kernel.
N=$(nvidia-smi -L | wc -l)
make -s -C paper_2406_14088_b200/csrc >/dev/null
timeout 900 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -1
for args in "llama7b_tp8_dp8_roundtrip --overlap on" "llama7b_tp8_dp8_roundtrip --overlap on --kernel 0" "llama7b_replicate_to_dp8 --mode relay" "llama7b_replicate_to_dp8 --mode relay --kernel 0"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $N --workload $args --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/q.log 2>&1
  echo "$args rc=$? $(tail -1 gpurun_out/q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["verified"])' 2>&1 | tail -1)"
done
