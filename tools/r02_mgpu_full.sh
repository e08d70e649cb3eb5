#!/bin/bash
# Full multi-GPU pytest (cross-GPU parity incl. multicast + full-size 7B, oversubscribed cases) with per-case lines.
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_build_mg_n$N.log 2>&1 || exit 1
timeout 2400 python -m pytest tests/test_multigpu.py -x -q -rP --durations=10 > gpurun_out/r02_pytest_multigpu_n$N.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/r02_pytest_multigpu_n$N.log; grep -c "^case .*: ok" gpurun_out/r02_pytest_multigpu_n$N.log; grep "FAIL" gpurun_out/r02_pytest_multigpu_n$N.log | head
