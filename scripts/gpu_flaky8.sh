#!/bin/bash
OUT=gpurun_out/${TAG:-flaky8}; mkdir -p $OUT
for i in 1 2 3 4 5 6; do
  timeout 600 python scripts/m4repro2.py 4000000 nocorpus > $OUT/r$i.log 2>&1
  echo "run $i: illegal=$(grep -c illegal $OUT/r$i.log) $(tr '\n' '|' < $OUT/r$i.log | cut -c1-200)" >> $OUT/flaky.log
done
for i in 1 2 3; do
  timeout 600 python -m pytest tests/test_gpu.py::test_solve_batch_c1_lanes tests/test_multi.py -m gpu -x -q > $OUT/p.log 2>&1
  echo "pytest run $i: $(tail -1 $OUT/p.log)" >> $OUT/flaky.log
done
for i in 1 2 3; do timeout 300 python scripts/solve_once.py tests/golden/c1/c1_S200_100001.scn 5 2>&1 | grep objective >> $OUT/flaky.log; done
