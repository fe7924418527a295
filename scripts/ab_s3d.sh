#!/bin/bash
mkdir -p gpurun_out
T=${1:-s3d}
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
C=gather_cfg1,gather_planned_cfg1
for g in tma flat; do RFL_GATHER=$g timeout 300 python scripts/kbench.py --graph --cases $C > gpurun_out/kb_${T}_$g.jsonl 2>&1; done
RFL_GATHER=jobs timeout 300 python scripts/kbench.py --graph --cases gather_cfg1 > gpurun_out/kb_${T}_jobs.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_csr_copy_tma" -s 3 -c 1 -o gpurun_out/prof_tma_$T -f python scripts/kbench.py --cases gather_planned_cfg1 --steps 3 --warmup 3 > gpurun_out/ncu_tma_$T.log 2>&1
RFL_TRACE=1 timeout 900 python scripts/shuffle_bench.py --ref-rows 0 > gpurun_out/shuffle_$T.json 2> gpurun_out/shuffle_$T.err
echo done
