#!/bin/bash
OUT=gpurun_out/${TAG:-minb}; mkdir -p $OUT
C1=tests/golden/c1/c1_S200_100001.scn
echo "default(6) $(timeout 300 python scripts/solve_once.py $C1 5 2>&1 | grep objective)" >> $OUT/minb.log
for B in 4 5 8; do
  echo "minb$B $(MGS_LIB_PATH=paper_2407_13126_b200/lib/variants/minb$B.so timeout 300 python scripts/solve_once.py $C1 5 2>&1 | grep objective)" >> $OUT/minb.log
  echo "minb$B lanes $(MGS_LIB_PATH=paper_2407_13126_b200/lib/variants/minb$B.so MGS_BATCH_LANES=8 timeout 300 python scripts/batch_probe.py 16 2>&1 | tail -1)" >> $OUT/minb.log
done
