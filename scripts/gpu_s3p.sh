#!/bin/bash
mkdir -p gpurun_out
T=${1:-s3p}
RIFFLE_E2E_TRACE=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
C=densify_cfg1,densify_bf16_cfg1,densify_norm_cfg2
for v in default v10:256:80:16:2 v10:256:40:8:3; do
  echo "== $v" >> gpurun_out/kb_${T}_densify.txt
  if [ $v = default ]; then timeout 300 python scripts/kbench.py --graph --cases $C >> gpurun_out/kb_${T}_densify.txt 2>&1
  else RFL_DENSIFY=$v timeout 300 python scripts/kbench.py --graph --cases $C >> gpurun_out/kb_${T}_densify.txt 2>&1; fi
done
timeout 600 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2_$T.json 2>&1
echo done
