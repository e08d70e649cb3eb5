#!/bin/bash
# Copy-engine relay piece size on the replicate workload at N GPUs, against the SM relay.
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
PORT=29600
for p in sm 64 128 512 1024; do
  PORT=$((PORT+1))
  if [ $p = sm ]; then opt="--ce-transport off"; else opt="--ce-transport on"; fi
  RR_RELAY_PIECE_MIB=$p timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $PORT \
    bench.py --gpus $N --workload llama7b_replicate_to_dp8 --mode relay $opt --probe off --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/q.log 2>&1
  echo "n=$N piece=$p rc=$? $(tail -1 gpurun_out/q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["verified"], d["executor"]["ce_transport_phases"])' 2>&1 | tail -1)"
done | tee gpurun_out/r02_relay_piece_sweep_n$N.txt
