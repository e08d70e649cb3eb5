#!/bin/bash
# Item claim order x write window on the default 1-GPU workload.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for rep in 1 2; do
for order in rr seq; do
for w in 16 64 0; do
  r=$(RR_ITEM_ORDER=$order RR_WRITE_WINDOW_MIB=$w timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1)
  echo "order=$order window=${w}MiB $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["roofline"]["achieved"], d["roofline"]["frac"], d["verified"], d["host_ms"])')"
done; done; done | tee gpurun_out/r02_order_sweep_n1.txt
