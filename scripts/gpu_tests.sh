#!/bin/bash
OUT=gpurun_out/${TAG:-tests}; mkdir -p $OUT
timeout ${T:-900} python -m pytest tests -m gpu -x -q ${ARGS} > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
