timeout 900 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/s2_pytest_mgpu.log 2>&1; echo pytest rc=$? >> gpurun_out/s2_pytest_mgpu.log
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/s2_bench_n$N.json 2> gpurun_out/s2_bench_n$N.err; echo bench rc=$? >> gpurun_out/s2_bench_n$N.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus $N --steps 3 --warmup 1 > gpurun_out/s2_ref_n$N.json 2> gpurun_out/s2_ref_n$N.err; echo ref rc=$? >> gpurun_out/s2_ref_n$N.err
