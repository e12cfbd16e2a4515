#!/bin/bash
# single-window C1 device time under launch-shape variants (tuning probe)
OUT=gpurun_out/${TAG:-grid}; mkdir -p $OUT
C1=tests/golden/c1/c1_S200_100001.scn
for CAP in 0 1 2 3 4 6; do
  echo "GRID_CAP=$CAP $(MGS_GRID_CAP=$CAP timeout 300 python scripts/solve_once.py $C1 5 2>&1 | grep objective)" >> $OUT/grid.log
done
echo "NO_FORK $(MGS_NO_FORK=1 timeout 300 python scripts/solve_once.py $C1 5 2>&1 | grep objective)" >> $OUT/grid.log
