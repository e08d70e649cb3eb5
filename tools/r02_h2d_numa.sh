#!/bin/bash
# Host link per GPU at N GPUs: concurrent pinned H2D with and without NUMA binding; topology.
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
{ nvidia-smi topo -m; lscpu | grep -i "numa\|socket\|model name"; free -g; } > gpurun_out/r02_topo_n$N.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29650 \
  tools/h2d_numa.py 4 2>&1 | tail -3 | tee gpurun_out/r02_h2d_numa_n$N.json
