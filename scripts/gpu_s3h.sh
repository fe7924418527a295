#!/bin/bash
mkdir -p gpurun_out
T=${1:-s3h}
df -h /tmp > gpurun_out/df_$T.txt
timeout 600 python bench.py --workload cfg5 > gpurun_out/bench_cfg5_$T.json 2> gpurun_out/bench_cfg5_$T.err; echo "rc=$?" >> gpurun_out/bench_cfg5_$T.err
df -h /tmp >> gpurun_out/df_$T.txt
rm -rf /tmp/riffle_bench/cfg5*
RIFFLE_E2E_TRACE=1 timeout 600 python bench.py --workload cfg4 --no-cpu-baseline > gpurun_out/bench_cfg4_$T.json 2> gpurun_out/bench_cfg4_$T.err; echo "rc=$?" >> gpurun_out/bench_cfg4_$T.err
rm -rf /tmp/riffle_bench/cfg4
bash scripts/ab_densify9.sh $T
echo done
