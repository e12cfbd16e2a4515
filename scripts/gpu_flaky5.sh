#!/bin/bash
OUT=gpurun_out/${TAG:-flaky5}; mkdir -p $OUT
for args in "4000000" "4000000 nocorpus" "8000000"; do
  for i in 1 2 3; do
    echo "[$args] run $i: $(timeout 600 python scripts/m4repro2.py $args 2>&1 | tr '\n' '|')" >> $OUT/flaky.log
  done
done
