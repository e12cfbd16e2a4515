#!/bin/bash
# The round-end driver's commands, as it runs them
OUT=gpurun_out/${TAG:-drv}; mkdir -p $OUT
( time python -m pytest tests/ -x -q -m gpu ) > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
( time python -c "import __graft_entry__ as g; g.smoke()" ) > $OUT/smoke.log 2>&1; echo "rc $?" >> $OUT/smoke.log
( time python bench.py ) > $OUT/bench.json 2> $OUT/bench.err; echo "rc $?" >> $OUT/bench.err
( time python bench.py --impl reference ) > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "rc $?" >> $OUT/bench_ref.err
