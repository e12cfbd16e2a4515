#!/bin/bash
OUT=gpurun_out/dbg7; mkdir -p $OUT
timeout 60 env MGS_TRACE=1 python -u scripts/solve_once.py tests/golden/kat/worked_example.scn > $OUT/trace.log 2>&1
