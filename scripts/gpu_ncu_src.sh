#!/bin/bash
# per-source-line stall samples (ncu --set full --import-source, -lineinfo build) of DP phase kernels at step ${STEP:-100}
OUT=gpurun_out/${TAG:-ncu_src}; mkdir -p $OUT
C1=tests/golden/c1/c1_S200_100001.scn
for K in ${KERNELS:-k_units k_scans k_tables k_trans_small k_write}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$K\b" --launch-skip ${STEP:-100} --launch-count 1 \
    -o $OUT/$K python scripts/solve_once.py $C1 1 > $OUT/$K.log 2>&1
  python scripts/ncu_hot.py $OUT/$K.ncu-rep 40 > $OUT/${K}_hot.txt 2>&1
  rm -f $OUT/$K.ncu-rep
done
