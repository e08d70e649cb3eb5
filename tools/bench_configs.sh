#!/bin/bash
# Bench every BASELINE.json workload that fits the GPUs of this box.
# 1 GPU: plain python; N GPUs: torchrun. Writes gpurun_out/configs_n$N.jsonl.
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
N=$(nvidia-smi -L | wc -l)
WORKLOADS=${WORKLOADS:-"tiny_tp2_to_dp2 llama7b_tp8_dp8_roundtrip llama7b_replicate_to_dp8 llama13b_pp2tp4_to_dp2tp4 llama34b_critic_pp4tp2_to_tp8 llama70b_pp2tp4_to_tp8"}
: > "$OUT/configs_n$N.jsonl"
for w in $WORKLOADS; do
  if [ "$w" = "llama70b_pp2tp4_to_tp8" ] && [ "$N" = "1" ]; then continue; fi  # 282 GB > one GPU
  if [ "$w" = "tiny_tp2_to_dp2" ] && [ "$N" != "1" ] && [ "$N" != "2" ]; then continue; fi
  if [ "$N" = "1" ]; then
    timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu > "$OUT/cfg_${w}_n$N.log" 2>&1
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29512 bench.py --gpus $N --workload $w --steps 10 --warmup 3 --no-e2e \
      > "$OUT/cfg_${w}_n$N.log" 2>&1
  fi
  echo "$w rc=$?"
  tail -1 "$OUT/cfg_${w}_n$N.log" >> "$OUT/configs_n$N.jsonl"
done
python - "$OUT/configs_n$N.jsonl" <<'PY'
import json, sys
for line in open(sys.argv[1]):
    try:
        d = json.loads(line)
    except Exception:
        print("unparsable:", line[:200]); continue
    r = d["roofline"]
    print(f'{d["config"]["workload"]:34s} N={d["n_gpus"]} ms={d["ms_per_step"]:.3f} phases={d["phase_ms"]} '
          f'{r["bound"]} {r["achieved"]} GB/s frac={r["frac"]} verified={d["verified"]}')
PY
