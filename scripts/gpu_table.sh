#!/bin/bash
OUT=gpurun_out/${TAG:-table}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu.py -m gpu -x -q -k "table" > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --batch 0 > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_table --launch-skip 2 --launch-count 1 -o $OUT/ncu_k_table python scripts/table_probe.py 4096 > $OUT/ncu.log 2>&1
