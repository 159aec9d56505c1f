#!/bin/bash
# Round evidence on one B200 (run through gpurun): the default bench line,
# the reference (CPU) arm, the ncu launch list of a short bench and one full
# ncu capture of the dominant kernel on the bench workload (C4).
#   tools/round_evidence.sh OUTDIR
set -o pipefail
OUT=${1:-gpurun_out/ev}
mkdir -p "$OUT"
timeout 900 python bench.py > "$OUT/bench.log" 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > "$OUT/ref.log" 2>&1; echo "ref rc=$?"
SHORT="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --cpu-seconds 0 --train-steps 0 --bf16-steps 0"
timeout 600 $SHORT > "$OUT/plain.log" 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file "$OUT/launches.csv" $SHORT > "$OUT/ncu_launches.log" 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:${2:-k_rotate_in}" -c 1 \
  -o "$OUT/prof_top" -f python bench.py --steps 1 --warmup 0 --e2e-steps 0 --cpu-seconds 0 --train-steps 0 --bf16-steps 0 \
  > "$OUT/ncu_full.log" 2>&1; echo "full rc=$?"
