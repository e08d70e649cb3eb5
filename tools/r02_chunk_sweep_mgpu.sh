#!/bin/bash
# Explicit work-item size on the default 7B workload at N GPUs (flag-synchronised phases use it as slot size too).
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
PORT=29500
for c in ${CHUNKS:-256 128 64 32}; do
  PORT=$((PORT+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $PORT \
    bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --no-cpu --chunk-kib $c --probe off ${EXTRA:-} > gpurun_out/q.log 2>&1
  echo "n=$N chunk=$c rc=$? $(tail -1 gpurun_out/q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["roofline"]["bound"], d["roofline"]["achieved"], d["verified"], d["host_ms"])' 2>&1 | tail -1)"
done | tee gpurun_out/r02_chunk_sweep_n$N.txt
