#!/bin/bash
# Staged gather (copy-engine rotation + per-piece unpack) vs the default path, 7B round trip at 2 and N GPUs.
OUT=${OUT:-gpurun_out}; mkdir -p $OUT
N=$(nvidia-smi -L | wc -l)
for w in $N 2; do
  for st in on off; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port 2965$w \
      bench.py --gpus $w --steps 10 --warmup 3 --no-e2e --staged $st $( [ $st = on ] && echo --overlap off ) ${EXTRA} 2>$OUT/staged_${w}_$st.err | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'n': d['n_gpus'], 'staged': '$st', 'phases': d['config']['staged_phases'], 'ms': d['ms_per_step'], 'phase_ms': d['phase_ms'], 'nvlink': d['nvlink_gbs_per_gpu'], 'verified': d['verified']}))" || tail -5 $OUT/staged_${w}_$st.err
  done
done
