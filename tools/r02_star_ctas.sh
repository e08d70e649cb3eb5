#!/bin/bash
# Do spinning fan-out CTAs slow the copy engines? CE star (7B) and CE relay (replicate) at N GPUs vs CTA count.
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
PORT=29700
for w in "llama7b_tp8_dp8_roundtrip --staged off --ce-transport on" "llama7b_replicate_to_dp8 --mode relay --ce-transport on"; do
  for c in 0 296 148 74; do
    PORT=$((PORT+1))
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $PORT \
      bench.py --gpus $N --workload $w --probe off --ctas $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/q.log 2>&1
    echo "n=$N $w ctas=$c rc=$? $(tail -1 gpurun_out/q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["executor"]; print(d["ms_per_step"], d["phase_ms"], d["verified"], e["ce_transport_phases"], e["relay_phases"], e["overlap_phases"])' 2>&1 | tail -1)"
  done
done | tee gpurun_out/r02_star_ctas_n$N.txt
