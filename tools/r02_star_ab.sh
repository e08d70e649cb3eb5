#!/bin/bash
# 7B tp8->dp8 at N GPUs: copy-engine star vs copy-engine transport (separate fan-out) vs staged, phase times.
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
PORT=29800
for opt in "--staged off --ce-transport on --probe off" "--staged off --ce-transport on --overlap off --probe off" "--staged on --probe off"; do
  PORT=$((PORT+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $PORT \
    bench.py --gpus $N --workload llama7b_tp8_dp8_roundtrip $opt --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/q.log 2>&1
  echo "n=$N $opt rc=$? $(tail -1 gpurun_out/q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["executor"]; print(d["ms_per_step"], d["phase_ms"], d["roofline"]["bound"], d["roofline"]["achieved"], d["verified"], "ce", e["ce_transport_phases"], "staged", e["staged_phases"], "ovl", e["overlap_phases"])' 2>&1 | tail -1)"
done | tee gpurun_out/r02_star_ab_n$N.txt
