#!/bin/bash
OUT=gpurun_out/dbg6; mkdir -p $OUT
timeout 120 env MGS_DEBUG_STEPS=1 python -u scripts/solve_once.py > $OUT/steps.log 2>&1
