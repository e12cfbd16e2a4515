#!/bin/bash
# Per-step device time of one C1 window (eager launches with events; serialised) + counters
OUT=gpurun_out/${TAG:-steps}; mkdir -p $OUT
timeout 300 env MGS_DEBUG_STEPS=1 MGS_STEP_TIMES=1 python -u scripts/solve_once.py ${SCN:-tests/golden/c1/c1_S200_100001.scn} 2 > $OUT/steps.log 2>&1; echo "rc $?" >> $OUT/steps.log
timeout 300 python -u scripts/solve_once.py ${SCN:-tests/golden/c1/c1_S200_100001.scn} 5 > $OUT/graph.log 2>&1; echo "rc $?" >> $OUT/graph.log
