#!/bin/bash
# Final multi-GPU evidence on N GPUs: default bench line (e2e included) at N and 2, the full multi-GPU pytest
# (cross-GPU world 2/N incl. multicast and full-size 7B, world 8 with two ranks per GPU when N = 4), and the
# 8-rank bench oversubscribed on N GPUs (correctness of the N=8 path, probe included).
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_build_final_n$N.log 2>&1 || exit 1
for G in 2 $N; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port $((29400+G)) \
    bench.py --gpus $G > gpurun_out/r02_bench_default_n$G.json 2> gpurun_out/r02_bench_default_n$G.err
  echo "bench n=$G rc=$?"; tail -c 600 gpurun_out/r02_bench_default_n$G.json; echo
done
timeout 2700 python -m pytest tests/test_multigpu.py -q -rP --durations=10 > gpurun_out/r02_pytest_multigpu_n$N.log 2>&1
echo "pytest multigpu rc=$?"; tail -4 gpurun_out/r02_pytest_multigpu_n$N.log; grep -c "^case .*: ok" gpurun_out/r02_pytest_multigpu_n$N.log; grep "FAIL" gpurun_out/r02_pytest_multigpu_n$N.log | head -5
if [ "$N" = 4 ]; then
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29488 \
    bench.py --gpus 8 --steps 3 --warmup 3 --no-cpu > gpurun_out/r02_bench_world8_on_4gpus.json 2> gpurun_out/r02_bench_world8_on_4gpus.err
  echo "bench world8 rc=$?"; tail -c 1500 gpurun_out/r02_bench_world8_on_4gpus.json
fi
