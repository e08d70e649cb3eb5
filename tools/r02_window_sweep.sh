#!/bin/bash
# Write-window sweep of the default 1-GPU workload (library-default item sizes, RR_WRITE_WINDOW_MIB).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for rep in 1 2; do
for w in ${WINDOWS:-0 8 16 32 64 128}; do
  r=$(RR_WRITE_WINDOW_MIB=$w timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1)
  echo "window=${w}MiB $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["roofline"]["achieved"], d["roofline"]["frac"], d["verified"])')"
done
done | tee gpurun_out/r02_window_sweep_n1.txt
