#!/bin/bash
# kD8Int8 value kind: staging / fused tests, cfg2 bench (counts); cfg3 / cfg4 lines over 200 steps
O=gpurun_out/s3n; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_staging.py tests/test_gpu_shapes.py -x -q > $O/pytest_staging.log 2>&1; echo "exit $?" >> $O/pytest_staging.log
timeout 600 python bench.py --workload cfg4 --steps 200 --warmup 10 --no-file-e2e > $O/bench_cfg4_k200.json 2> $O/bench_cfg4_k200.err
timeout 600 python bench.py --workload cfg3 --steps 200 --warmup 10 --no-file-e2e > $O/bench_cfg3_k200.json 2> $O/bench_cfg3_k200.err
timeout 1800 python bench.py --workload cfg2 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
