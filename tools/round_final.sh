#!/bin/bash
# End-of-round evidence on one B200 (through gpurun): the GPU test suite,
# smoke(), then tools/round_evidence.sh (default bench line, reference arm,
# ncu launch list, one full ncu capture of the dominant kernel).
#   tools/round_final.sh OUTDIR
set -o pipefail
OUT=${1:-gpurun_out/final}
mkdir -p "$OUT"
timeout 1200 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"
bash tools/round_evidence.sh "$OUT"
