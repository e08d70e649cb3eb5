#!/bin/bash
# chunk / CTA sweep of the default 1-GPU workload
for c in 256 128 64 32 16; do
  for ctas in 0 148 296; do
    r=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --chunk-kib $c --ctas $ctas 2>/dev/null | tail -1)
    echo "chunk=$c ctas=$ctas $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["roofline"]["achieved"], d["verified"])')"
  done
done
