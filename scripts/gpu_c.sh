# fused densify-from-delta-records: parity + cfg2 / cfg1 loader numbers + launch list
mkdir -p gpurun_out
T=${1:-c}
timeout 600 python -m pytest tests/test_gpu_staging.py -x -q --timeout 300 > gpurun_out/pytest_staging_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_staging_$T.log
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$T.log
RIFFLE_PROC_ROWS=500000 timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-file-e2e > gpurun_out/bench_cfg2s_$T.json 2> gpurun_out/bench_$T.err
RFL_FUSED=0 RIFFLE_PROC_ROWS=500000 timeout 900 python bench.py --workload cfg2 --no-cpu-baseline --no-file-e2e > gpurun_out/bench_cfg2s_nofuse_$T.json 2>> gpurun_out/bench_$T.err
timeout 600 python bench.py --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > gpurun_out/bench_$T.json 2>> gpurun_out/bench_$T.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > /dev/null 2>&1
