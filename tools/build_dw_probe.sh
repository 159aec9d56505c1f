#!/bin/sh
# Builds tools/bin/dw_probe (the tensor-core dW kernel against a host sum).
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/bin
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_2507_03840_b200/csrc \
  -o tools/bin/dw_probe tools/dw_probe.cu -Lpaper_2507_03840_b200 -lesg_b200 \
  -Xlinker -rpath='$ORIGIN/../../paper_2507_03840_b200' -Xlinker -rpath=/usr/lib/x86_64-linux-gnu
