#!/bin/bash
# Default bench line, reference arm and ncu launch list at N=1 (driver-style), with wall time and peak RSS.
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/r02_build_b1.log 2>&1 || { tail -20 $OUT/r02_build_b1.log; exit 1; }
free -g > $OUT/r02_bench_n1_mem.txt
python tools/run_measured.py python bench.py > $OUT/r02_bench_n1.json 2> $OUT/r02_bench_n1.err; echo "b200 rc=$?"
tail -1 $OUT/r02_bench_n1.err
python tools/run_measured.py python bench.py --impl reference > $OUT/r02_bench_ref_n1.json 2> $OUT/r02_bench_ref_n1.err; echo "ref rc=$?"
tail -1 $OUT/r02_bench_ref_n1.err
tail -c 3000 $OUT/r02_bench_n1.json; echo; tail -c 1500 $OUT/r02_bench_ref_n1.json; echo
if [ "${NCU:-1}" = 1 ]; then
  LIST_CMD="python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1"
  $LIST_CMD > $OUT/r02_plain_list.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/r02_launches_n1.csv \
        $LIST_CMD > $OUT/r02_ncu_list.log 2>&1
  echo "launch list rc=$?"
fi
