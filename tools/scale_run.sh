set -o pipefail
mkdir -p gpurun_out/scale2
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500+N)) bench.py --gpus $N --steps 3 --warmup 3 --e2e-steps 1 --cpu-seconds 0 > gpurun_out/scale2/scale_$N.log 2>&1
  echo "N=$N rc=$?"
done
