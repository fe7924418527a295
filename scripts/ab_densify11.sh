#!/bin/bash
# densify A/B: v9 default vs v11 (TMA-staged row entries) + a correctness pass of v11
mkdir -p gpurun_out
T=${1:-s3u}
RFL_DENSIFY=v11:256:72:8:2 timeout 600 python -m pytest tests/test_gpu_loader.py tests/test_gpu_fullsize.py -x -q -k "densify or normalize or bf16 or fullsize or cfg1" > gpurun_out/pytest_v11_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v11_$T.log
C=densify_cfg1,densify_bf16_cfg1,densify_norm_cfg2
for v in default v11:256:72:8:2 v11:256:40:8:3 v11:256:80:8:2 v11:256:64:8:2 v11:256:100:16:1; do
  echo "== $v" >> gpurun_out/kb_${T}_densify.txt
  if [ $v = default ]; then timeout 300 python scripts/kbench.py --graph --cases $C >> gpurun_out/kb_${T}_densify.txt 2>&1
  else RFL_DENSIFY=$v timeout 300 python scripts/kbench.py --graph --cases $C >> gpurun_out/kb_${T}_densify.txt 2>&1; fi
done
echo done
