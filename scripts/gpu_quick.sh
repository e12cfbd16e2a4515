#!/bin/bash
# quick perf check of the C1 window: eager per-kernel split + graph timing (+ optional tests)
OUT=gpurun_out/${TAG:-quick}; mkdir -p $OUT
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests/test_gpu.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log; fi
{
for V in "" ${VARIANTS}; do
echo "=== variant [$V] eager"; timeout 120 env $V MGS_DEBUG_STEPS=1 python -u scripts/solve_once.py 2>&1 | grep "in-stream"
echo "=== variant [$V] graph x5"; timeout 120 env $V python -u scripts/solve_once.py tests/golden/c1/c1_S200_100001.scn 5 2>&1 | grep objective
done
MGS_BATCH_LANES=8 timeout 300 python scripts/batch_probe.py 16 2>&1 | tail -1
} > $OUT/quick.log 2>&1
