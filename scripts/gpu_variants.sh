#!/bin/bash
# C1 device time and 16-window lane batches for each library variant in lib/variants (tuning probe)
OUT=gpurun_out/${TAG:-variants}; mkdir -p $OUT
C1=tests/golden/c1/c1_S200_100001.scn
echo "default $(timeout 300 python scripts/solve_once.py $C1 5 2>&1 | grep objective)" >> $OUT/variants.log
for V in paper_2407_13126_b200/lib/variants/*.so; do
  echo "$(basename $V) $(MGS_LIB_PATH=$V timeout 300 python scripts/solve_once.py $C1 5 2>&1 | grep objective)" >> $OUT/variants.log
  echo "$(basename $V) $(MGS_LIB_PATH=$V MGS_BATCH_LANES=8 timeout 300 python scripts/batch_probe.py 16 2>&1 | tail -1)" >> $OUT/variants.log
done
