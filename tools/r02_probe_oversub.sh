set -x
mkdir -p gpurun_out
( nproc; free -g; lscpu | grep -i "model name\|^CPU(s)\|Socket\|NUMA node(s)"; nvidia-smi -L ) > gpurun_out/r02_box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for W in 2 4; do
  start=$(date +%s)
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$W --master-addr=127.0.0.1 --master-port=2950$W tests/dist_worker.py > gpurun_out/r02_oversub_w$W.log 2>&1
  echo "world $W rc=$? secs=$(( $(date +%s) - start ))" >> gpurun_out/r02_box.txt
done
tail -3 gpurun_out/r02_oversub_w*.log
cat gpurun_out/r02_box.txt
