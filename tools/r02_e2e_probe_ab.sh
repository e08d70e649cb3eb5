#!/bin/bash
# e2e at N GPUs: default line (probe, auto/multicast-allocated sets) vs probe off, same box; host-link probe first.
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29650 \
  tools/h2d_numa.py 4 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("h2d concurrent", [round(r["unbound_concurrent"],1) for r in d["gbs"]], "alone", [round(r["unbound_alone"],1) for r in d["gbs"]])'
PORT=29780
for opts in "" "--probe off --staged on" "--probe off --staged on --mode mc" "" ; do
  PORT=$((PORT+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $PORT \
    bench.py --gpus $N $opts --steps 5 --warmup 3 --e2e-steps 5 --no-cpu > gpurun_out/q.log 2>&1
  echo "n=$N [$opts] rc=$? $(tail -1 gpurun_out/q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["executor"]; print(d["ms_per_step"], d["phase_ms"], "e2e", d["e2e"]["ms_per_step"], d["e2e"]["value"], d["verified"], e.get("staged_phases"), e.get("multicast_sets"))' 2>&1 | tail -1)"
done 2>&1 | tee gpurun_out/r02_e2e_probe_ab_n$N.txt
