#!/bin/bash
# Round-end scaling evidence on one box with 4 GPUs (run through gpurun --gpus 4):
# forward strong scaling (bench.py, C4) at 1/2/4 GPUs and config-5 training
# weak scaling (tools/train_bench.py --config C5) at 1/2/4 GPUs.
set -o pipefail
OUT=${1:-gpurun_out/scale}
mkdir -p "$OUT"
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-seconds 0 --train-steps 0 --bf16-steps 0 \
  > "$OUT/fwd_n1.log" 2>&1; echo "fwd N=1 rc=$?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500+N)) bench.py --gpus $N --steps 3 --warmup 3 --cpu-seconds 0 \
    --train-steps 0 --bf16-steps 0 > "$OUT/fwd_n$N.log" 2>&1; echo "fwd N=$N rc=$?"
done
timeout 900 python tools/train_bench.py --config C5 --steps 2 > "$OUT/c5_n1.log" 2>&1; echo "c5 N=1 rc=$?"
for N in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29800+N)) tools/train_bench.py --config C5 --steps 2 > "$OUT/c5_n$N.log" 2>&1
  echo "c5 N=$N rc=$?"
done
