#!/bin/bash
# Multi-GPU evidence run (needs >= 4 GPUs): C3 partitioned forward at 2 and 4
# GPUs bit-exact against the serial forward, C2 at 4 GPUs with the serial
# heads also against the float oracle (the oracle's C3 forward takes too long
# for one call), the multi-GPU pytest cases, and the C4 bench at N = 2 and 4.
# Logs go to gpurun_out/multi/.
OUT=gpurun_out/multi
mkdir -p $OUT
nvidia-smi -L > $OUT/gpus.txt; nproc >> $OUT/gpus.txt; free -g >> $OUT/gpus.txt
for W in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
    --master-port $((29500 + W)) tools/multi_gpu_check.py --config C3 --golden > $OUT/c3_w$W.log 2>&1
  echo "c3 w$W rc=$?" >> $OUT/rc.txt
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29510 tools/multi_gpu_check.py --config C2 --oracle > $OUT/c2_w4.log 2>&1
echo "c2 w4 rc=$?" >> $OUT/rc.txt
timeout 900 python -m pytest tests/test_gpu_multi.py -q > $OUT/pytest_multi.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + N)) bench.py --gpus $N --steps 5 --warmup 3 --train-steps 0 > $OUT/bench_n$N.log 2>&1
  echo "bench n$N rc=$?" >> $OUT/rc.txt
done
