#!/bin/bash
mkdir -p gpurun_out
T=${1:-s3m}
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$T.json 2>&1
for c in 16 32 64 128; do RFL_PULL=1 RFL_PULL_CTAS=$c timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_pull${c}_$T.json 2>&1; done
rm -rf /tmp/riffle_bench/cfg1
for w in cfg3 cfg4; do timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_${w}_$T.json 2>&1; rm -rf /tmp/riffle_bench/$w; done
echo done
