#!/bin/bash
# Long multi-GPU fuzz (tests/dist_worker.py, fuzz section) with several seeds:
# random placement pairs x delivery options (push/pull, flat/hierarchical,
# relay, overlap, staged gather, copy-engine runs and transport, kernels, item
# sizes, normal and special-value weights), each launched twice, bit-exact
# against the oracle. One `case ...: ok <s>` line per case in the logs.
OUT=${OUT:-gpurun_out}; mkdir -p $OUT
N=$(nvidia-smi -L | wc -l)
CASES=${CASES:-150}
for seed in ${SEEDS:-11 12}; do
  for w in 2 $N; do
    RR_SECTIONS=fuzz RR_FUZZ_SEED=$seed RR_FUZZ_CASES=$CASES timeout 1500 python -m torch.distributed.run --nnodes=1 \
      --nproc-per-node $w --master-addr 127.0.0.1 --master-port $((29600 + seed + w)) tests/dist_worker.py \
      > $OUT/fuzz_w${w}_s$seed.log 2>&1
    echo "world=$w seed=$seed cases=$CASES rc=$? ok=$(grep -c '^case .*: ok' $OUT/fuzz_w${w}_s$seed.log) fail=$(grep -c '^case .*: FAIL' $OUT/fuzz_w${w}_s$seed.log) $(tail -1 $OUT/fuzz_w${w}_s$seed.log)"
  done
done
