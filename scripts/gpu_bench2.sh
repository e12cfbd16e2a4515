#!/bin/bash
# bench N=1 (default legs) + a functional 2-rank run sharing one GPU over gloo
OUT=gpurun_out/${TAG:-bench2}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 900 python bench.py ${BENCH_ARGS} > $OUT/bench.json 2> $OUT/bench.err; echo "rc $?" >> $OUT/bench.err
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 3 --warmup 3 --batch 4 > $OUT/bench_g2.json 2> $OUT/bench_g2.err; echo "rc $?" >> $OUT/bench_g2.err
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log; fi
