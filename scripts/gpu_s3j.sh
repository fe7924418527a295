#!/bin/bash
mkdir -p gpurun_out
T=${1:-s3j}
C=densify_cfg1,densify_bf16_cfg1,densify_norm_cfg2
for v in default v9:256:64:8:3 v9:256:72:8:3 v9:128:72:16:3 v9:128:52:16:4 v9:128:36:8:6 v9:512:100:4:2 v9:256:100:16:2; do
  echo "== $v" >> gpurun_out/kb_${T}_densify.txt
  if [ $v = default ]; then timeout 300 python scripts/kbench.py --graph --cases $C >> gpurun_out/kb_${T}_densify.txt 2>&1
  else RFL_DENSIFY=$v timeout 300 python scripts/kbench.py --graph --cases $C >> gpurun_out/kb_${T}_densify.txt 2>&1; fi
done
timeout 300 python scripts/pcie_calib.py > gpurun_out/pcie_$T.json 2>&1
RIFFLE_E2E_TRACE=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_trace_$T.json 2> gpurun_out/bench_trace_$T.err
rm -rf /tmp/riffle_bench/kb_cfg1 /tmp/riffle_bench/kb_cfg2s
KB_FULL=1 timeout 900 python scripts/kbench.py --graph --cases dense_bf16_cfg3,dense_raw_cfg4 > gpurun_out/kb_${T}_full.jsonl 2>&1
echo done
