#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) on the smoke (tiny config: LDG/STG kernel,
# TMA bulk ring with special values, barrier kernel) and on a small 1-GPU parity subset.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/r02_sanitizer_smoke_$tool.log 2>&1
  echo "smoke $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/r02_sanitizer_smoke_$tool.log | tail -1)"
done
for tool in memcheck racecheck; do
  timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest -q -x tests/test_gpu_parity.py \
    -k "reinterleave_bitexact and 0-1 or special_value_words_2byte or spec_tiny_unaligned" \
    > gpurun_out/r02_sanitizer_parity_$tool.log 2>&1
  echo "parity $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/r02_sanitizer_parity_$tool.log | tail -2 | tr '\n' ' ')"
done
