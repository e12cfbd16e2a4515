#!/bin/bash
OUT=gpurun_out/${TAG:-flaky}; mkdir -p $OUT
for V in paper_2407_13126_b200/lib/variants/*.so; do
  for i in 1 2 3 4; do
    MGS_LIB_PATH=$V timeout 600 python -m pytest tests/test_gpu.py tests/test_multi.py -m gpu -x -q > $OUT/p.log 2>&1
    echo "$(basename $V) run $i: $(tail -1 $OUT/p.log) $(grep -h -o "CUDA error[^']*" $OUT/p.log | head -1)" >> $OUT/flaky.log
  done
done
