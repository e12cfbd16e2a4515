#!/bin/bash
OUT=gpurun_out/${TAG:-flaky4}; mkdir -p $OUT
for mode in "MGS_SER_RS=1" "MGS_SER_TRANS=1" "MGS_SER_RANK=1"; do
  for i in 1 2 3; do
    env $mode timeout 600 python -m pytest tests/test_gpu.py::test_solve_batch_c1_lanes tests/test_multi.py -m gpu -x -q > $OUT/p.log 2>&1
    echo "[$mode] run $i: $(tail -1 $OUT/p.log) $(grep -h -o "CUDA error[^']*" $OUT/p.log | head -1)" >> $OUT/flaky.log
  done
done
