#!/bin/bash
mkdir -p gpurun_out
T=${1:-s3k}
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
RFL_PACK=warp timeout 300 python scripts/kbench.py --graph --cases pack_cfg5 > gpurun_out/kb_${T}_pack.jsonl 2>&1
timeout 300 python scripts/kbench.py --graph --cases pack_cfg5 >> gpurun_out/kb_${T}_pack.jsonl 2>&1
for n in 1 2; do RFL_H2D_STREAMS=$n timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_h2d${n}_$T.json 2>&1; done
rm -rf /tmp/riffle_bench/cfg1
timeout 600 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/bench_cfg5_$T.json 2>&1
echo done
