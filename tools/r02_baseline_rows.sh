#!/bin/bash
# BASELINE.md's per-N rows (one plan device per GPU) with the default bench (probe on): 2-GPU rows on GPUs 0-1.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
PORT=29200
for f in examples/baseline_rows/*.json; do
  g=$(python -c "import json,sys; print(json.load(open('$f'))['cluster']['gpus_per_node'])")
  vis=$(python -c "print(','.join(str(i) for i in range($g)))")
  PORT=$((PORT+1))
  CUDA_VISIBLE_DEVICES=$vis timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 \
    --master-port $PORT bench.py --gpus $g --config $f --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/q.log 2>&1
  echo "rc=$? $f" >&2
  tail -1 gpurun_out/q.log
done > gpurun_out/r02_baseline_rows.jsonl
python - <<'PY'
import json
for ln in open("gpurun_out/r02_baseline_rows.jsonl"):
    try: d = json.loads(ln)
    except Exception: print("bad", ln[:300]); continue
    r = d["roofline"]; e = d["executor"]
    print(d["config"]["workload"], d["n_gpus"], d["ms_per_step"], r["bound"], r["achieved"], r["frac"], d["verified"],
          [(p["chosen"], p["ms"]) for p in e["policy_probe"]])
PY
