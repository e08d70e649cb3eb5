#!/bin/bash
# Round-2 GPU check: build, smoke, pytest -m gpu (verbose, per-case lines), on however many GPUs the box has.
# Usage: bash tools/r02_gpu_check.sh [tag] [pytest args...]
TAG=${1:-n1}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_build_$TAG.log 2>&1 || { tail -30 gpurun_out/r02_build_$TAG.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_$TAG.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/r02_smoke_$TAG.log
timeout 3000 python -m pytest tests -m gpu -x -q -rA --durations=25 "$@" > gpurun_out/r02_pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/r02_pytest_gpu_$TAG.log
