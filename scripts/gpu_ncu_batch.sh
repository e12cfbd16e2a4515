#!/bin/bash
# ncu --set full of the DP phase kernels at step ~100 of a 32-lane C1 batch (throughput mode)
OUT=gpurun_out/${TAG:-ncu_batch}; mkdir -p $OUT
DP='regex:k_(kid_scan|kid_fill|ranks_small|ranks_big|units|scans|trans_small|tables|trans_big|band|write|dom)\b'
MGS_BATCH_LANES=32 timeout 300 python scripts/batch_probe.py ${N:-32} > $OUT/batch_time.log 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none -k "$DP" --launch-skip ${SKIP:-1200} --launch-count 13 \
  -o $OUT/ncu_batch python scripts/batch_probe.py ${N:-32} > $OUT/ncu_batch.log 2>&1; echo "rc $?" >> $OUT/ncu_batch.log
if [ -f $OUT/ncu_batch.ncu-rep ]; then
  ncu -i $OUT/ncu_batch.ncu-rep --page raw --csv > $OUT/ncu_batch_raw.csv 2>/dev/null; gzip -f $OUT/ncu_batch_raw.csv
  python scripts/ncu_hot.py $OUT/ncu_batch.ncu-rep 60 > $OUT/ncu_batch_hot.txt 2>&1
  rm -f $OUT/ncu_batch.ncu-rep
fi
