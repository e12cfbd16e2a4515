#!/bin/bash
OUT=gpurun_out/${TAG:-multi}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
# functional N=2 check of bench.py's torchrun path (both ranks share the one GPU; gloo collectives)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --batch 0 --table 0 > $OUT/bench2.json 2> $OUT/bench2.err; echo "rc $?" >> $OUT/bench2.err
