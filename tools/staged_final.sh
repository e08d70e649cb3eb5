#!/bin/bash
# Staged gather: multi-GPU parity (incl. 8 ranks on 4 GPUs) and the default bench (staged auto) at 4 and 2 GPUs.
OUT=${OUT:-gpurun_out}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > $OUT/staged_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/staged_pytest.log
for w in 4 2; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port 2967$w \
    bench.py --gpus $w > $OUT/staged_bench_n$w.json 2>$OUT/staged_bench_n$w.err
  python -c "import json; d=json.loads(open('$OUT/staged_bench_n$w.json').read().strip().splitlines()[-1]); print($w, d['ms_per_step'], d['phase_ms'], d['config']['staged_phases'], d['config']['overlap_phases'], d['e2e']['value'], d['e2e'].get('verified'), d['verified'], d['gpu_launches'])"
done
