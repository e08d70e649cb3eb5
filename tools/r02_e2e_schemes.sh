#!/bin/bash
# e2e (sources onloaded from pinned host memory) per delivery scheme at N GPUs.
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
PORT=29760
for opts in "--probe off --staged on" "--probe off --staged off" "--probe off --staged off --overlap off" "--probe off --staged off --mode relay" "--probe off --staged off --ce-transport on"; do
  PORT=$((PORT+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $PORT \
    bench.py --gpus $N $opts --steps 5 --warmup 3 --e2e-steps 5 --no-cpu > gpurun_out/q.log 2>&1
  echo "n=$N $opts rc=$? $(tail -1 gpurun_out/q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], "e2e", d["e2e"]["ms_per_step"], d["e2e"]["value"], d["verified"])' 2>&1 | tail -1)"
done | tee gpurun_out/r02_e2e_schemes_n$N.txt
