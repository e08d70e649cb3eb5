#!/bin/bash
# Copy-engine sweep on the default 1-GPU workload (no e2e / CPU legs).
# Usage: bash tools/sweep_kernels.sh [extra bench args]
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
# the ring shapes swept in round 1 (2-4, 6-16) were pruned from the library; see profiles/r01_sweep_kernels*.txt
for k in ${KERNELS:-0 1 5}; do
  line=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --kernel $k "$@" 2>/dev/null | tail -1)
  echo "kernel=$k $(echo "$line" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["roofline"]["achieved"], d["roofline"]["frac"], d["verified"])' 2>&1)"
done | tee "$OUT/sweep_kernels.txt"
