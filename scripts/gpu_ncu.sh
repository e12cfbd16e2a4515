#!/bin/bash
# ncu --set full of selected kernels of the C1 window. NCU_KERNELS, NCU_SKIP
OUT=gpurun_out/${TAG:-ncu}; mkdir -p $OUT
for K in ${NCU_KERNELS}; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$K\b" --launch-skip ${NCU_SKIP:-300} --launch-count 1 \
  -o $OUT/ncu_${K}_s${NCU_SKIP:-300} python scripts/solve_once.py tests/golden/c1/c1_S200_100001.scn 1 > $OUT/ncu_$K.log 2>&1; echo "rc $?" >> $OUT/ncu_$K.log
done
