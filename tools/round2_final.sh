#!/bin/bash
# Final round-2 check on one B200 (gpurun): GPU test suite, smoke, the
# driver's bench command and the reference arm.  Logs in OUTDIR.
OUT=${1:-gpurun_out/r02final}
mkdir -p "$OUT"
nvidia-smi -L > "$OUT/gpu.txt"; nproc >> "$OUT/gpu.txt"
timeout 1500 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/rc.txt"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/rc.txt"
timeout 900 python bench.py --steps 20 --warmup 5 > "$OUT/bench.log" 2>&1; echo "bench rc=$?" >> "$OUT/rc.txt"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > "$OUT/ref.log" 2>&1; echo "ref rc=$?" >> "$OUT/rc.txt"
