#!/bin/bash
# Fuzz at world 8 on a 4-GPU box (two ranks per GPU): the 8-rank code path with random delivery options.
OUT=${OUT:-gpurun_out/r02fuzz}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for seed in ${SEEDS:-81 82}; do
  RR_SECTIONS=fuzz RR_FUZZ_SEED=$seed RR_FUZZ_CASES=${CASES:-100} timeout 2400 python -m torch.distributed.run --nnodes=1 \
    --nproc-per-node 8 --master-addr 127.0.0.1 --master-port $((29500 + seed)) tests/dist_worker.py \
    > $OUT/fuzz_w8_on4_s$seed.log 2>&1
  echo "world=8 (on 4 GPUs) seed=$seed rc=$? ok=$(grep -c '^case .*: ok' $OUT/fuzz_w8_on4_s$seed.log) fail=$(grep -c '^case .*: FAIL' $OUT/fuzz_w8_on4_s$seed.log) $(tail -1 $OUT/fuzz_w8_on4_s$seed.log)"
done
