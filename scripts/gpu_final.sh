#!/bin/bash
# round-end style pass: GPU tests, smoke, bench N=1, a 2-rank gloo bench on one GPU, ncu of the non-DP kernels
OUT=gpurun_out/${TAG:-final}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q --durations=12 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?" >> $OUT/bench.err
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 3 --warmup 3 --batch 4 > $OUT/bench_g2.json 2> $OUT/bench_g2.err; echo "rc $?" >> $OUT/bench_g2.err
if [ -n "$NCU" ]; then
timeout 1800 ncu --set full --import-source on --clock-control none \
  -k 'regex:\bk_(?!(kids|kid_scan|kid_fill|ranks_small|ranks_big|units|scans|place|trans_small|tables|trans_big|band|write|dom)\b)' \
  --launch-count 90 -o $OUT/ncu_other python scripts/exercise_all.py > $OUT/ncu_other.log 2>&1; echo "rc $?" >> $OUT/ncu_other.log
if [ -f $OUT/ncu_other.ncu-rep ]; then
  ncu -i $OUT/ncu_other.ncu-rep --page raw --csv > $OUT/ncu_other_raw.csv 2>/dev/null; gzip -f $OUT/ncu_other_raw.csv; rm -f $OUT/ncu_other.ncu-rep
fi
fi
du -sh $OUT
