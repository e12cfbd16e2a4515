#!/bin/bash
OUT=gpurun_out/dbg8; mkdir -p $OUT
for T in 1024 512 256 128; do echo "threads $T"; MGS_GREEDY_THREADS=$T python scripts/solve_once.py tests/golden/c1/c1_S200_100001.scn 3 2>&1 | tail -2; done > $OUT/greedy.log 2>&1
