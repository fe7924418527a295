#!/bin/bash
# Full evidence pass on one B200: GPU tests, smoke, bench lines for every workload
# (stores removed after use: /tmp is ~80 GB), reference arm, kernel table, launch
# list and one ncu --set full capture of the default bench's densify kernel.
# Usage: bash scripts/gpu_round.sh <tag>
mkdir -p gpurun_out
T=${1:-r1}
B=/tmp/riffle_bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$T.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
timeout 600 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2>> gpurun_out/bench_$T.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv \
   python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_densify -s 3 -c 1 \
   -o gpurun_out/prof_densify_$T -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$T.log 2>&1
rm -rf $B/cfg1
for w in cfg5 cfg2 cfg3 cfg4; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_${w}_$T.json 2>> gpurun_out/bench_$T.err
  rm -rf $B/${w}*
done
timeout 900 python scripts/kbench.py --graph > gpurun_out/kbench_$T.jsonl 2>&1
echo done
