#!/bin/bash
# kD8IntP: parity (staging / shapes / loader tests), cfg2 e2e, cfg1 e2e unchanged
O=gpurun_out/s3q; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_staging.py tests/test_gpu_shapes.py tests/test_gpu_loader.py -x -q > $O/pytest_intp.log 2>&1; echo "exit $?" >> $O/pytest_intp.log
timeout 1800 python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 python bench.py --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > $O/bench_cfg1.json 2> $O/bench_cfg1.err
