#!/bin/bash
# auto multicast is a probe-only candidate: parity of the multicast / probe sections, and the default lines with and without the probe.
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
RR_SECTIONS=multicast,probe timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29931 tests/dist_worker.py > gpurun_out/r02_mc_auto_n$N.log 2>&1
echo "dist n=$N rc=$? ok=$(grep -c '^case .*: ok' gpurun_out/r02_mc_auto_n$N.log) fail=$(grep -c '^case .*: FAIL' gpurun_out/r02_mc_auto_n$N.log) $(tail -1 gpurun_out/r02_mc_auto_n$N.log)"
PORT=29940
for opts in "" "--probe off"; do
  PORT=$((PORT+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $PORT \
    bench.py --gpus $N $opts --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/q.log 2>&1
  echo "n=$N [$opts] rc=$? $(tail -1 gpurun_out/q.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["executor"]; print(d["ms_per_step"], d["phase_ms"], d["verified"], "mc", e["multicast_sets"], "staged", e["staged_phases"], "ovl", e["overlap_phases"], e["policy_probe"])' 2>&1 | tail -1)"
done
