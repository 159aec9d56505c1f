#!/bin/bash
# Full ncu capture of the first N kernel launches of a short C2 forward
# (run on the GPU box, after the same bench command has passed without ncu).
#   tools/prof.sh NAME [N] [REGEX]  -> gpurun_out/NAME.ncu-rep
set -eo pipefail
NAME=${1:?name}; N=${2:-8}; RE=${3:-.}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$RE" -c "$N" \
  -o "gpurun_out/$NAME" -f python bench.py --config C2 --steps 1 --warmup 0 --e2e-steps 0 --cpu-seconds 0 \
  > "gpurun_out/$NAME.log" 2>&1
