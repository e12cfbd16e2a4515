#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench, launch list, ncu captures. Output -> gpurun_out/$TAG
OUT=gpurun_out/${TAG:-run}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/smi.txt 2>&1
{ nproc; lscpu | grep 'Model name'; } > $OUT/host.txt
if [ -z "$SKIP_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?" >> $OUT/smoke.log
fi
timeout 900 python bench.py ${BENCH_ARGS} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?" >> $OUT/bench.err
if [ -n "$REF" ]; then
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "rc $?" >> $OUT/bench_ref.err
fi
if [ -n "$NCU" ]; then
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python scripts/solve_once.py tests/golden/c1/c1_S200_100001.scn 2 > $OUT/ncu_launches.log 2>&1; echo "rc $?" >> $OUT/ncu_launches.log
for K in ${NCU_KERNELS:-k_trans_big k_write}; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K --launch-skip ${NCU_SKIP:-300} --launch-count 1 \
  -o $OUT/ncu_$K python scripts/solve_once.py tests/golden/c1/c1_S200_100001.scn 2 > $OUT/ncu_$K.log 2>&1; echo "rc $?" >> $OUT/ncu_$K.log
done
fi
