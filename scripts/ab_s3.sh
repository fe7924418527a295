#!/bin/bash
# A/B for the balanced CSR copy + PDL (session 3): tests, kbench graph with PDL off/on, legacy gather.
mkdir -p gpurun_out
T=${1:-s3c}
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
C=gather_cfg1,gather_planned_cfg1,dense_bf16_cfg3,dense_raw_cfg4,densify_cfg1,densify_norm_cfg2
RFL_GATHER=jobs timeout 300 python scripts/kbench.py --graph --cases gather_cfg1 > gpurun_out/kb_${T}_legacy.jsonl 2>&1
RFL_PDL=0 timeout 600 python scripts/kbench.py --graph --cases $C > gpurun_out/kb_${T}_pdl0.jsonl 2>&1
RFL_PDL=1 timeout 600 python scripts/kbench.py --graph --cases $C > gpurun_out/kb_${T}_pdl1.jsonl 2>&1
RFL_PDL=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_${T}_pdl0.json 2>&1
RFL_PDL=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_${T}_pdl1.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_csr_copy_flat" -s 3 -c 1 -o gpurun_out/prof_flat_$T -f python scripts/kbench.py --cases gather_planned_cfg1 --steps 3 --warmup 3 > gpurun_out/ncu_flat_$T.log 2>&1
echo done
