#!/bin/bash
OUT=gpurun_out/${TAG:-lanes2}; mkdir -p $OUT
for L in 8 16; do for SH in 0 2 4; do
  echo "lanes $L share $SH: $(MGS_LANE_SHARE=$SH MGS_BATCH_LANES=$L timeout 300 python scripts/batch_probe.py 32 2>&1 | tail -1)" >> $OUT/lanes.log
done; done
