#!/bin/bash
# ncu --set full of the kernels the first "other" capture's launch cap did not reach
OUT=gpurun_out/${TAG:-ncu_rest}; mkdir -p $OUT
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k 'regex:\bk_(replay|bruteforce|bruteforce_final|table|weight_caps|pareto_flag|views|check|eval_views|fluid|greedy_one)\b' \
  --launch-count 20 -o $OUT/ncu_rest python scripts/exercise_all.py > $OUT/ncu_rest.log 2>&1; echo "rc $?" >> $OUT/ncu_rest.log
if [ -f $OUT/ncu_rest.ncu-rep ]; then
  ncu -i $OUT/ncu_rest.ncu-rep --page raw --csv > $OUT/ncu_rest_raw.csv 2>/dev/null; gzip -f $OUT/ncu_rest_raw.csv; rm -f $OUT/ncu_rest.ncu-rep
fi
