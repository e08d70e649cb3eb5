timeout 900 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/pytest_mgpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_mgpu.log
N=$(nvidia-smi -L | wc -l)
for k in 1 0; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 --kernel $k --no-e2e > gpurun_out/bench_n${N}_k$k.log 2>&1; echo bench k=$k rc=$?
tail -1 gpurun_out/bench_n${N}_k$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["phase_ms"], d["nvlink_gbs_per_gpu"], d["roofline"], d["verified"])'
done
