#!/bin/bash
# Builds tools/bin/so2_probe (development timing probe for k_so2_tc).
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$R/tools/bin"
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr \
  -I/usr/include "$R/tools/so2_probe.cu" -o "$R/tools/bin/so2_probe"
