#!/bin/bash
mkdir -p gpurun_out
T=${1:-s3n}
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q --timeout 600 > gpurun_out/pytest_full_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full_$T.log
timeout 900 python -m pytest tests -x -q -m gpu --timeout 600 > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
for s in 0:256 2:256 3:256; do echo "== $s" >> gpurun_out/kb_${T}_dg.txt; RFL_DG=$s timeout 300 python scripts/kbench.py --graph --cases dense_bf16_cfg3,dense_raw_cfg4 >> gpurun_out/kb_${T}_dg.txt 2>&1; done
for w in cfg3 cfg4; do timeout 900 python bench.py --workload $w > gpurun_out/bench_${w}_$T.json 2>&1; rm -rf /tmp/riffle_bench/$w; done
echo done
