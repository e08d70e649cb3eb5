for ctas in 8 16 32 64 148 0; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29577 \
    bench.py --gpus 2 --workload llama13b_pp2tp4_to_dp2tp4 --steps 5 --warmup 3 --no-e2e --ce on --ctas $ctas 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ctas=$ctas', d['ms_per_step'], d['phase_ms'], d['verified'])"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 tools/ce_ipc_probe.py 2>&1 | tail -1
