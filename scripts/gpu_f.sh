mkdir -p gpurun_out
T=${1:-f}
timeout 600 python -m pytest tests/test_gpu_staging.py -x -q --timeout 300 > gpurun_out/pytest_staging_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_staging_$T.log
timeout 900 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/bench_cfg5_$T.json 2> gpurun_out/bench_$T.err
RFL_PACK_ISOLATE=1 timeout 900 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/bench_cfg5_iso_$T.json 2>> gpurun_out/bench_$T.err
RFL_TRACE=1 timeout 900 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/bench_cfg5_tr_$T.json 2> gpurun_out/trace_cfg5_$T.err
