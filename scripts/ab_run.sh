#!/bin/bash
# A/B pass: full GPU tests, HBM calibration, densify-variant parity, densify variant sweep.
mkdir -p gpurun_out
T=${1:-ab}
if [ -n "$FULL_TESTS" ]; then
  timeout 900 python -m pytest tests -q -m gpu -x --timeout 180 > gpurun_out/pytest_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$T.log
fi
timeout 300 python scripts/hbm_calib.py > gpurun_out/hbm_$T.json 2>&1
for V in ${PARITY_VARIANTS:-}; do
  echo "## parity $V" >> gpurun_out/parity_$T.log
  RFL_DENSIFY=$V timeout 300 python -m pytest tests -x -q -m gpu --timeout 120 -k "densify or normalize or bf16 or golden" >> gpurun_out/parity_$T.log 2>&1
done
VARIANTS=${VARIANTS:-"v2:256:40"} bash scripts/ab_densify.sh > gpurun_out/ab_$T.txt 2>&1
