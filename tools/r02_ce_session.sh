#!/bin/bash
# Copy-engine transport session on N GPUs: probe, parity, A/B bench per config.
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_build_ce_n$N.log 2>&1 || { tail -30 gpurun_out/r02_build_ce_n$N.log; exit 1; }
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/ce2d_probe tools/ce2d_probe.cu
[ "$N" -ge 2 ] && timeout 600 tools/ce2d_probe > gpurun_out/r02_ce2d_probe_n$N.txt 2>&1
cat gpurun_out/r02_ce2d_probe_n$N.txt
PORT=29600
for w in llama70b_pp2tp4_to_tp8 llama34b_critic_pp4tp2_to_tp8 llama13b_pp2tp4_to_dp2tp4 llama7b_tp8_dp8_roundtrip; do
  for opt in "--ce-transport on --probe off" "--ce-transport off --probe off" "--probe on"; do
    PORT=$((PORT+1))
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $PORT \
      bench.py --gpus $N --workload $w $opt --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/q.log 2>&1
    echo "n=$N $w $opt rc=$? $(tail -1 gpurun_out/q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["executor"]; print(d["ms_per_step"], d["phase_ms"], d["nvlink_gbs_per_gpu"], d["roofline"]["achieved"], d["roofline"]["frac"], d["verified"], "ce", e["ce_transport_phases"], "staged", e["staged_phases"], "ovl", e["overlap_phases"], "probe", e["policy_probe"], d["host_ms"])' 2>&1 | tail -1)"
  done
done | tee gpurun_out/r02_ce_ab_n$N.txt
if [ "${PARITY:-1}" = 1 ]; then
  RR_SECTIONS=${SECTIONS:-cetransport,probe,basic,staged,fuzz} timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29690 tests/dist_worker.py > gpurun_out/r02_dist_ce_n$N.log 2>&1
  echo "dist rc=$?"; grep -c "^case" gpurun_out/r02_dist_ce_n$N.log; grep "FAIL\|rank .*:\|world=" gpurun_out/r02_dist_ce_n$N.log | head -20
fi
