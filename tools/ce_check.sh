#!/bin/bash
# Copy-engine runs: multi-GPU parity (pytest + fuzz with CE forced on small
# ranges) and the stage-remap config with CE on/off at 2 and N GPUs.
OUT=${OUT:-gpurun_out}; mkdir -p $OUT; P=${P:-ce2}
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > $OUT/${P}_pytest_mgpu.log 2>&1; echo "pytest rc=$?"
CASES=200 SEEDS="31" OUT=$OUT/${P}_fuzz bash tools/fuzz_long.sh
grep -h "copy-engine" $OUT/${P}_fuzz/*.log
: > $OUT/${P}_bench.jsonl
for w in 2 $N; do
  for ce in on off; do
    for wl in llama13b_pp2tp4_to_dp2tp4 llama7b_tp8_dp8_roundtrip; do
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port 29577 \
        bench.py --gpus $w --workload $wl --steps 10 --warmup 3 --no-e2e --ce $ce 2>/dev/null | tail -1 >> $OUT/${P}_bench.jsonl
    done
  done
done
python - $OUT/${P}_bench.jsonl <<'PY'
import json, sys
for l in open(sys.argv[1]):
    try: d = json.loads(l)
    except Exception: print("bad line", l[:200]); continue
    print(d["config"]["workload"], d["n_gpus"], d["config"].get("ce_runs"), d["ms_per_step"], d["phase_ms"], d["nvlink_gbs_per_gpu"], d["verified"])
PY
