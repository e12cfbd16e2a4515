#!/bin/bash
OUT=gpurun_out/${TAG:-quick2}; mkdir -p $OUT
{
for L in 1 8; do
echo "=== lanes $L eager"; MGS_DEBUG_STEPS=1 MGS_BATCH_LANES=$L timeout 300 python scripts/batch_probe.py $L 2>&1 | grep -E "in-stream|lanes="
done
} > $OUT/quick.log 2>&1
