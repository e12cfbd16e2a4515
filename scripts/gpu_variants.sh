#!/bin/bash
# A/B of prebuilt library variants (paper_2407_13126_b200/lib/variants/*.so): C1 device time + eager per-kernel times
OUT=gpurun_out/${TAG:-variants}; mkdir -p $OUT
C1=tests/golden/c1/c1_S200_100001.scn
L=paper_2407_13126_b200/lib
for v in ${VARIANTS:-base A B}; do
  cp $L/variants/$v.so $L/libmigsim_b200.so
  for r in 1 2; do echo "$v $(timeout 300 python scripts/solve_once.py $C1 5 2>&1 | grep objective)" >> $OUT/time.log; done
  echo "$v $(MGS_DEBUG_STEPS=1 timeout 300 python scripts/solve_once.py $C1 1 2>&1 | grep in-stream)" >> $OUT/time.log
  echo "$v $(MGS_BATCH_LANES=16 timeout 300 python scripts/batch_probe.py 16 2>&1 | tail -1)" >> $OUT/time.log
done
