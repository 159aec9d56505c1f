#!/bin/bash
# Config 5 weak scaling of the training step on 2 and 4 GPUs (tools/train_bench.py --config C5)
set -o pipefail
mkdir -p gpurun_out/train_scale
for N in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29800+N)) tools/train_bench.py --config C5 --steps 2 > gpurun_out/train_scale/c5_n$N.log 2>&1
  echo "N=$N rc=$?"; tail -1 gpurun_out/train_scale/c5_n$N.log
done
