#!/bin/bash
# NVLink hardware counters (NVML) around fixed-scheme bench runs: payload vs wire bytes of copy-engine transport vs SM stores.
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
PORT=29900
for w in llama70b_pp2tp4_to_tp8 llama34b_critic_pp4tp2_to_tp8; do
  for opt in "--ce-transport on" "--ce-transport off --ce off --staged off"; do
    PORT=$((PORT+1))
    python tools/nvlink_nvml.py -- python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $PORT bench.py --gpus $N --workload $w $opt --probe off --steps 10 --warmup 3 --no-e2e --no-cpu \
      > gpurun_out/q_nv.log 2> gpurun_out/q_nv.err
    echo "$w $opt :: $(grep '^{"metric' gpurun_out/q_nv.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["algorithmic_bytes_per_launch"], d["executor"]["ce_transport_phases"])') :: $(tail -1 gpurun_out/q_nv.log)"
  done
done | tee gpurun_out/r02_nvlink_counters_n$N.txt
