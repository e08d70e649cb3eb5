#!/bin/bash
# NCCL send/recv + local unpack vs this library (copy-engine runs) on the 13B stage remap, 2 and N GPUs.
OUT=${OUT:-gpurun_out}; mkdir -p $OUT
N=$(nvidia-smi -L | wc -l)
for w in 2 $N; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port 2962$w \
    tools/nccl_compare.py --workload llama13b_pp2tp4_to_dp2tp4 --kind p2p 2>/dev/null | tail -1
  for ce in on off; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port 2963$w \
      bench.py --gpus $w --workload llama13b_pp2tp4_to_dp2tp4 --steps 10 --warmup 3 --no-e2e --ce $ce 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'impl': 'b200', 'ce': '$ce', 'n_gpus': d['n_gpus'], 'ms': d['ms_per_step'], 'phase_ms': d['phase_ms'], 'verified': d['verified']}))"
  done
done
