#!/bin/bash
# Where does the copy-engine relay lose time against the bare chain (tools/ce_relay_probe.cu)?
# Replicate workload at N GPUs: overlap on/off (in-host fan-out concurrent or after), CTA count, piece size.
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
PORT=29870
run() {  # env, opts
  PORT=$((PORT+1))
  env $1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $PORT \
    bench.py --gpus $N --workload llama7b_replicate_to_dp8 --probe off --steps 10 --warmup 3 --no-e2e --no-cpu $2 > gpurun_out/q.log 2>&1
  echo "[$1] [$2] rc=$? $(tail -1 gpurun_out/q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["executor"]; print(d["ms_per_step"], d["phase_ms"], d["verified"], "relay", e["relay_phases"], "ce", e["ce_transport_phases"], "ovl", e["overlap_phases"])' 2>&1 | tail -1)"
}
{
run "X=1" "--mode relay --ce-transport on"
run "X=1" "--mode relay --ce-transport on --overlap off"
run "X=1" "--mode relay --ce-transport on --ctas 148"
run "RR_RELAY_PIECE_MIB=128" "--mode relay --ce-transport on --ctas 148"
run "RR_RELAY_PIECE_MIB=192" "--mode relay --ce-transport on --ctas 148"
run "X=1" "--mode relay --ce-transport off"
run "X=1" "--mode relay --ce-transport off --overlap off"
} | tee gpurun_out/r02_relay_decomp_n$N.txt
