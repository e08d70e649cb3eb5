#!/bin/bash
# NVLink-bound phase sweep (7B tp8->dp8, N GPUs): mode x copy kernel x CTAs.
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
N=$(nvidia-smi -L | wc -l)
for mode in push pull; do
  for k in 1 0 5; do
    for c in 0 148 296; do
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port 29517 bench.py --gpus $N --mode $mode --kernel $k --ctas $c --steps 10 --warmup 3 \
        --no-e2e > "$OUT/nvl_${mode}_${k}_${c}.log" 2>&1
      echo "mode=$mode kernel=$k ctas=$c $(tail -1 "$OUT/nvl_${mode}_${k}_${c}.log" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["roofline"]["achieved"], d["verified"])' 2>&1 | tail -1)"
    done
  done
done | tee "$OUT/nvlink_sweep_n$N.txt"
