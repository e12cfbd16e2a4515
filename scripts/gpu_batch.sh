#!/bin/bash
OUT=gpurun_out/${TAG:-batch}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
{
for L in 1 2 4 8 16; do MGS_BATCH_LANES=$L timeout 300 python scripts/batch_probe.py 16 2>&1 | tail -2; done
} > $OUT/batch.log 2>&1
