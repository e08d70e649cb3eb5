#!/bin/bash
# CTA-count sweep of the multicast (multimem.st) path on the replicate workload.
OUT=${OUT:-gpurun_out}
N=$(nvidia-smi -L | wc -l)
for c in 74 148 296 444 592; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29516 bench.py --gpus $N --workload llama7b_replicate_to_dp8 --mode mc --ctas $c --steps 10 \
    --warmup 3 --no-e2e > "$OUT/mcctas_$c.log" 2>&1
  echo "ctas=$c rc=$? $(tail -1 "$OUT/mcctas_$c.log" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["verified"])' 2>&1 | tail -1)"
done | tee "$OUT/mc_ctas_n$N.txt"
