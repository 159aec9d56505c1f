#!/bin/bash
# 8-GPU evidence on one node (gpurun --gpus 8, or the driver's 8-GPU step):
# C3 partitioned forward at 8 ranks bit-exact against the serial forward and
# the committed float-oracle sample, then the C4 bench at N = 8 (the driver's
# own scaling run launches bench.py the same way).
OUT=gpurun_out/multi8
mkdir -p $OUT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
  --master-port 29508 tools/multi_gpu_check.py --config C3 --golden > $OUT/c3_w8.log 2>&1
echo "c3 w8 rc=$?" >> $OUT/rc.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
  --master-port 29608 bench.py --gpus 8 --steps 5 --warmup 3 --train-steps 0 > $OUT/bench_n8.log 2>&1
echo "bench n8 rc=$?" >> $OUT/rc.txt
