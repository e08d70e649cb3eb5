#!/bin/bash
# Every BASELINE config with the default bench (probe on) at N GPUs, plus the dist parity of the transport schemes.
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_build_cfg_n$N.log 2>&1 || exit 1
PORT=29700
for w in ${WORKLOADS:-llama7b_tp8_dp8_roundtrip llama13b_pp2tp4_to_dp2tp4 llama34b_critic_pp4tp2_to_tp8 llama70b_pp2tp4_to_tp8 llama7b_replicate_to_dp8}; do
  PORT=$((PORT+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $PORT \
    bench.py --gpus $N --workload $w --steps 10 --warmup 3 ${EXTRA:---no-e2e --no-cpu} > gpurun_out/q.log 2>&1
  echo "rc=$?" >&2
  tail -1 gpurun_out/q.log
done > gpurun_out/r02_configs_n$N.jsonl
python - <<PY
import json
for ln in open("gpurun_out/r02_configs_n$N.jsonl"):
    try: d=json.loads(ln)
    except Exception: print("bad line", ln[:200]); continue
    e=d["executor"]; r=d["roofline"]
    print(d["config"]["workload"], d["ms_per_step"], d["phase_ms"], "nvl", d["nvlink_gbs_per_gpu"], r["bound"], r["achieved"], r["frac"], d["verified"], [(p["chosen"], p["ms"]) for p in e["policy_probe"]])
PY
if [ "${PARITY:-0}" = 1 ]; then
  RR_SECTIONS=cetransport timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29790 tests/dist_worker.py > gpurun_out/r02_dist_cet_n$N.log 2>&1
  echo "dist rc=$?"; grep -c "^case" gpurun_out/r02_dist_cet_n$N.log; grep "FAIL\|rank .*:\|world=" gpurun_out/r02_dist_cet_n$N.log | head
fi
