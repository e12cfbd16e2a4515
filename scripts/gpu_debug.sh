#!/bin/bash
OUT=gpurun_out/dbg; mkdir -p $OUT
S=tests/golden/kat/worked_example.scn
C=tests/golden/c1/c1_S24_100004.scn
{
echo "=== v2 graph worked"; timeout 60 python -u scripts/solve_once.py $S 2>&1 | tail -5
echo "=== v2 graph c1s24 x3"; timeout 60 python -u scripts/solve_once.py $C 3 2>&1 | tail -5
echo "=== v2 eager c1s200"; timeout 120 env MGS_DEBUG_STEPS=1 python -u scripts/solve_once.py 2>&1 | grep -v "^v2 step" | tail -8
echo "=== v2 graph c1s200 x5"; timeout 120 python -u scripts/solve_once.py tests/golden/c1/c1_S200_100001.scn 5 2>&1 | tail -5
} > $OUT/triage3.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
