#!/bin/bash
# densify A/B: v6 default vs v9 (lane-parallel row lookups) vs v8 (un-scatter)
mkdir -p gpurun_out
T=${1:-s3g}
C=densify_cfg1,densify_bf16_cfg1,densify_norm_cfg2
for v in default v9:256:40:8:3 v9:256:40:8:4 v9:256:80:16:2 v8:256:40:8:3 v6:256:80:16:2; do
  echo "== $v" >> gpurun_out/kb_${T}_densify.txt
  if [ $v = default ]; then timeout 300 python scripts/kbench.py --graph --cases $C >> gpurun_out/kb_${T}_densify.txt 2>&1
  else RFL_DENSIFY=$v timeout 300 python scripts/kbench.py --graph --cases $C >> gpurun_out/kb_${T}_densify.txt 2>&1; fi
done
echo done
