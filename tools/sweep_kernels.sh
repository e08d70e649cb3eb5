#!/bin/bash
# Copy-engine sweep on the default 1-GPU workload (no e2e / CPU legs).
# Usage: bash tools/sweep_kernels.sh [extra bench args]
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
for k in ${KERNELS:-0 1 2 3 4 5 6 7 8 9 10}; do
  line=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --kernel $k "$@" 2>/dev/null | tail -1)
  echo "kernel=$k $(echo "$line" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["roofline"]["achieved"], d["roofline"]["frac"], d["verified"])' 2>&1)"
done | tee "$OUT/sweep_kernels.txt"
