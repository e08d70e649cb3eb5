#!/bin/bash
# Staged gather at N GPUs: piece size x SM CTA count (7B tp8->dp8 forward).
N=$(nvidia-smi -L | wc -l)
for mib in ${MIBS:-128 512 2048}; do
  for ctas in ${CTAS:-0 148}; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29661 \
      bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --staged on --overlap off --stage-mib $mib --ctas $ctas 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mib=$mib ctas=$ctas', d['ms_per_step'], d['phase_ms'], d['verified'])"
  done
done
