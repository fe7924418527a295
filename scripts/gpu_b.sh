mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mix_bw scripts/cuda/mix_bw.cu > /dev/null 2>&1
timeout 300 /tmp/mix_bw > gpurun_out/mix_bw_b.jsonl 2>&1
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_b.log
RIFFLE_PROC_ROWS=500000 timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-file-e2e > gpurun_out/bench_cfg2s_b.json 2> gpurun_out/bench_b.err
timeout 600 python bench.py --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > gpurun_out/bench_b.json 2>> gpurun_out/bench_b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > /dev/null 2>&1
