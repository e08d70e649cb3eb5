set -x
nvidia-smi -L > gpurun_out/s2_smi.txt
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/s2_pytest_mgpu_n4.log 2>&1; echo rc=$? >> gpurun_out/s2_pytest_mgpu_n4.log
for N in 4 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N > gpurun_out/s2_bench_n$N.json 2> gpurun_out/s2_bench_n$N.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --impl reference > gpurun_out/s2_bench_ref_n$N.json 2> gpurun_out/s2_bench_ref_n$N.err
done
