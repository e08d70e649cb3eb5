#!/bin/bash
# Copy-engine relay: parity (relay section, plus oversubscribed world 2/4 on GPU 0) and the replicate workload A/B.
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
RR_SECTIONS=relay timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29950 tests/dist_worker.py > gpurun_out/r02_relay_n$N.log 2>&1
echo "dist n=$N rc=$?"; grep -c "^case .*: ok" gpurun_out/r02_relay_n$N.log; grep "FAIL\|rank .*:\|world=" gpurun_out/r02_relay_n$N.log | head
for W in 2 4; do
  CUDA_VISIBLE_DEVICES=0 RR_SECTIONS=relay timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port $((29960+W)) tests/dist_worker.py > gpurun_out/r02_relay_oversub_w$W.log 2>&1
  echo "oversub w=$W rc=$?"; grep -c "^case .*: ok" gpurun_out/r02_relay_oversub_w$W.log; grep "FAIL\|rank .*:\|world=" gpurun_out/r02_relay_oversub_w$W.log | head -5
done
PORT=29970
for opt in "--mode relay --ce-transport off --probe off" "--mode relay --ce-transport on --probe off" "--probe on"; do
  PORT=$((PORT+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $PORT \
    bench.py --gpus $N --workload llama7b_replicate_to_dp8 $opt --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/q.log 2>&1
  echo "n=$N replicate $opt rc=$? $(tail -1 gpurun_out/q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["executor"]; print(d["ms_per_step"], d["phase_ms"], d["roofline"]["achieved"], d["verified"], "relay", e["relay_phases"], "ce", e["ce_transport_phases"], [(p["chosen"], p["ms"]) for p in e["policy_probe"]])' 2>&1 | tail -1)"
done | tee gpurun_out/r02_relay_ab_n$N.txt
