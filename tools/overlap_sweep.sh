#!/bin/bash
# Work-item (= flag) size x CTA count on the overlapped multi-GPU default bench.
N=$(nvidia-smi -L | wc -l)
for c in 128 256 512 1024; do
  for ctas in 0 444 296; do
    r=$(timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port 29551 bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --chunk-kib $c --ctas $ctas 2>/dev/null | tail -1)
    echo "n=$N chunk=$c ctas=$ctas $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["roofline"]["bound"], d["roofline"]["frac"], d["verified"])')"
  done
done
timeout 300 python bench.py --config examples/llama7b_train_gen_roundtrip.json --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | cut -c1-300
