#!/bin/bash
OUT=gpurun_out/${TAG:-lanes}; mkdir -p $OUT
for L in 4 8 12 16; do MGS_BATCH_LANES=$L timeout 300 python scripts/batch_probe.py 32 >> $OUT/lanes.log 2>&1; done
for B in 4 6 8; do MGS_MINB=$B echo "minb $B (build-time only)" >> $OUT/lanes.log; done
