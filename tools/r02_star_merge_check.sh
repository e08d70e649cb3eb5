#!/bin/bash
# Star pushes that also store the local destinations (one source read): parity and the 7B default line.
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for W in 2 $N; do
  RR_SECTIONS=basic,overlap,relay,probe,fuzz RR_FUZZ_CASES=120 RR_FUZZ_SEED=$((90+W)) timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port $((29920+W)) tests/dist_worker.py > gpurun_out/r02_star_merge_w$W.log 2>&1
  echo "dist w=$W rc=$? ok=$(grep -c '^case .*: ok' gpurun_out/r02_star_merge_w$W.log) fail=$(grep -c '^case .*: FAIL' gpurun_out/r02_star_merge_w$W.log) $(tail -1 gpurun_out/r02_star_merge_w$W.log)"
done
PORT=29930
for W in 2 $N; do
 for opts in "" "--staged off --probe off"; do
  PORT=$((PORT+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port $PORT \
    bench.py --gpus $W $opts --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/q.log 2>&1
  echo "n=$W [$opts] rc=$? $(tail -1 gpurun_out/q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["executor"]; r=d["roofline"]; print(d["ms_per_step"], d["phase_ms"], d["verified"], r["bound"], r["achieved"], r["frac"], r["algorithmic_bytes_per_launch"], "ovl", e["overlap_phases"], "staged", e["staged_phases"], [(p["chosen"], p["ms"]) for p in e["policy_probe"]])' 2>&1 | tail -1)"
 done
done
