#!/bin/sh
# Builds tools/bin/f16x3_probe (the fp16x3 chain with per-role wait accounting).
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/bin
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr \
  -Ipaper_2507_03840_b200/csrc -o tools/bin/f16x3_probe tools/f16x3_probe.cu -Xlinker -rpath=/usr/lib/x86_64-linux-gnu
