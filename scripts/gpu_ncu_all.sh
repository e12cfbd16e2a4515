#!/bin/bash
# ncu evidence for every kernel on the path (B200_PROFILING.md recipe; numbers taken under ncu are never bench values)
OUT=gpurun_out/${TAG:-ncu_all}; mkdir -p $OUT
C1=tests/golden/c1/c1_S200_100001.scn
# gpurun copies back <= 64 MiB: keep CSV exports (raw metrics + details), not the .ncu-rep files
export_rep() {
  if [ -f $1.ncu-rep ]; then
    ncu -i $1.ncu-rep --page raw --csv > $1_raw.csv 2>/dev/null
    ncu -i $1.ncu-rep --page details --csv > $1_details.csv 2>/dev/null
    gzip -f $1_raw.csv $1_details.csv
    rm -f $1.ncu-rep
  fi
}
DP='regex:k_(kids|kid_scan|kid_fill|ranks_small|ranks_big|units|scans|place|trans_small|tables|trans_big|band|write|dom)\b'
# 1. launch list of one C1 window: per-launch duration + DRAM bytes, cold (ncu flushes caches per kernel)
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches_cold.csv python scripts/solve_once.py $C1 1 > $OUT/launches_cold.log 2>&1; echo "rc $?" >> $OUT/launches_cold.log
gzip -f $OUT/launches_cold.csv
# 2. the same with --cache-control none (warm L2: live traffic of the window)
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv \
  --log-file $OUT/launches_warm.csv python scripts/solve_once.py $C1 1 > $OUT/launches_warm.log 2>&1; echo "rc $?" >> $OUT/launches_warm.log
gzip -f $OUT/launches_warm.csv
# 3. --set full of every DP phase kernel at the peak-frontier step (~100)
timeout 1800 ncu --set full --import-source on --clock-control none -k "$DP" --launch-skip ${DP_SKIP:-1300} --launch-count 13 \
  -o $OUT/ncu_dp_step100 python scripts/solve_once.py $C1 1 > $OUT/ncu_dp.log 2>&1; echo "rc $?" >> $OUT/ncu_dp.log
export_rep $OUT/ncu_dp_step100
# 4. --set full of every kernel outside the step loop (first launch of each); SKIP_OTHER=1 skips it
if [ -z "$SKIP_OTHER" ]; then
timeout 1800 ncu --set full --import-source on --clock-control none \
  -k 'regex:\bk_(?!(kids|kid_scan|kid_fill|ranks_small|ranks_big|units|scans|place|trans_small|tables|trans_big|band|write|dom)\b)' \
  --launch-count 80 -o $OUT/ncu_other python scripts/exercise_all.py > $OUT/ncu_other.log 2>&1; echo "rc $?" >> $OUT/ncu_other.log
export_rep $OUT/ncu_other
fi
du -sh $OUT
