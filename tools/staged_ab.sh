#!/bin/bash
# Same box, 4 GPUs: default bench with the staged gather (auto) vs without, e2e included; twice each.
for rep in 1 2; do
  for st in auto off; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29681 \
      bench.py --gpus 4 --staged $st 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('staged=$st', d['ms_per_step'], d['phase_ms'], 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], d['verified'])"
  done
done
