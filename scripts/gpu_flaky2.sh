#!/bin/bash
OUT=gpurun_out/${TAG:-flaky2}; mkdir -p $OUT
run() {
  for i in 1 2 3 4; do
    timeout 600 python -m pytest $@ -m gpu -x -q > $OUT/p.log 2>&1
    echo "[$*] run $i: $(tail -1 $OUT/p.log) $(grep -h -o "CUDA error[^']*" $OUT/p.log | head -1)" >> $OUT/flaky.log
  done
}
run tests/test_multi.py
run tests/test_gpu.py::test_solve_batch_c1_lanes tests/test_multi.py
run tests/test_gpu.py::test_solve_c1_fixtures tests/test_multi.py
run tests/test_gpu.py::test_solve_random_corpus tests/test_gpu.py::test_solve_batch_random_corpus tests/test_multi.py
