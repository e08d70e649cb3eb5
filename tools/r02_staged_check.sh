#!/bin/bash
# Staged gather with aligned rounds: parity (staged sections, N GPUs and world 2/4 on GPU 0) and the 7B A/B.
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
RR_SECTIONS=staged,fuzz RR_FUZZ_CASES=40 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29350 tests/dist_worker.py > gpurun_out/r02_staged_n$N.log 2>&1
echo "dist n=$N rc=$?"; grep -c "^case .*: ok" gpurun_out/r02_staged_n$N.log; grep "FAIL\|rank .*:\|world=" gpurun_out/r02_staged_n$N.log | head -5
for W in 2 4; do
  CUDA_VISIBLE_DEVICES=0 RR_SECTIONS=staged timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port $((29360+W)) tests/dist_worker.py > gpurun_out/r02_staged_oversub_w$W.log 2>&1
  echo "oversub w=$W rc=$?"; grep -c "^case .*: ok" gpurun_out/r02_staged_oversub_w$W.log; grep "FAIL\|rank .*:\|world=" gpurun_out/r02_staged_oversub_w$W.log | head -3
done
bash tools/r02_star_ab.sh
