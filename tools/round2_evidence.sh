#!/bin/bash
# Round-2 evidence on one B200 (run through gpurun): GPU test suite, smoke,
# the default bench line (fp32 headline), the reference arm, the ncu launch
# list of a short bench, and full ncu captures of the two dominant fp32
# kernels (layer-1 launches: -s 68 skips layer 0's 2 x 34 chunk launches).
#   tools/round2_evidence.sh OUTDIR
set -o pipefail
OUT=${1:-gpurun_out/r02}
mkdir -p "$OUT"
nvidia-smi -L > "$OUT/gpu.txt"; nproc >> "$OUT/gpu.txt"; free -g >> "$OUT/gpu.txt"
timeout 1500 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > "$OUT/bench.log" 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > "$OUT/ref.log" 2>&1; echo "ref rc=$?"
SHORT="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --cpu-seconds 0 --train-steps 0 --bf16-steps 0"
timeout 600 $SHORT > "$OUT/plain.log" 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file "$OUT/launches.csv" $SHORT > "$OUT/ncu_launches.log" 2>&1; echo "launches rc=$?"
ONE="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --cpu-seconds 0 --train-steps 0 --bf16-steps 0"
# layer-1 launches: -s skips layer 0's launches of the kernel (2 x 34 chunk
# launches for rotate_in / the chain, 34 for the node update)
for KS in "so2_f16x3 68" "k_rotate_in 68" "k_node_update 34"; do
  set -- $KS
  timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:$1" -s $2 -c 1 \
    -o "$OUT/prof_$1" -f $ONE > "$OUT/ncu_full_$1.log" 2>&1; echo "full $1 rc=$?"
done
# training step (C2): launch list of one step after a warm-up one
timeout 600 python tools/train_profile.py --steps 3 > "$OUT/train.log" 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/train_launches.csv" python tools/train_profile.py --steps 1 > "$OUT/ncu_train.log" 2>&1
echo "train rc=$?"
# chunking invariance and the tf32 cross-check at C3
timeout 600 python tools/f3_chunk_check.py --config C3 > "$OUT/chunk_c3.log" 2>&1; echo "chunk rc=$?"
