#!/bin/bash
OUT=gpurun_out/dbg4; mkdir -p $OUT
timeout 60 env MGS_TRACE=1 python -u scripts/chain_probe.py rnd_777_0 > $OUT/new_trace.log 2>&1
