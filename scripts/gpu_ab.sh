#!/bin/bash
# quick A/B: parity subset + C1 device time + 16-window lane batch
OUT=gpurun_out/${TAG:-ab}; mkdir -p $OUT
C1=tests/golden/c1/c1_S200_100001.scn
timeout 600 python -m pytest tests/test_gpu.py tests/test_multi.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
for r in 1 2; do timeout 300 python scripts/solve_once.py $C1 5 2>&1 | grep objective >> $OUT/time.log; done
MGS_BATCH_LANES=16 timeout 300 python scripts/batch_probe.py 16 >> $OUT/time.log 2>&1
${EXTRA:-true}
