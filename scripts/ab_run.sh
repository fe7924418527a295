#!/bin/bash
# A/B pass: HBM calibration, densify-variant parity, densify variant sweep.
mkdir -p gpurun_out
T=${1:-ab}
timeout 300 python scripts/hbm_calib.py > gpurun_out/hbm_$T.json 2>&1
for V in ${PARITY_VARIANTS:-v6:256:40:8:4}; do
  echo "## parity $V" >> gpurun_out/parity_$T.log
  RFL_DENSIFY=$V timeout 600 python -m pytest tests -x -q -m gpu -k "densify or normalize or bf16 or golden" >> gpurun_out/parity_$T.log 2>&1
done
VARIANTS=${VARIANTS:-"v2:256:40 v6:256:40:8:4"} bash scripts/ab_densify.sh > gpurun_out/ab_$T.txt 2>&1
