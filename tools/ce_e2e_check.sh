#!/bin/bash
# 13B stage remap with the e2e (onload) leg at 2 and 4 GPUs: copy-engine runs issued after the last onload chunk.
OUT=${OUT:-gpurun_out}; mkdir -p $OUT
for w in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port 2959$w \
    bench.py --gpus $w --workload llama13b_pp2tp4_to_dp2tp4 --steps 10 --warmup 3 2>$OUT/ce_e2e_n$w.err | tail -1 > $OUT/ce_e2e_n$w.json
  python -c "import json; d=json.load(open('$OUT/ce_e2e_n$w.json')); print($w, d['ms_per_step'], d['config']['ce_runs'], d['e2e'], d['verified'])"
done
