#!/bin/bash
# bit-packed column deltas in the pinned image: parity (staging / shapes / loader / deflate tests), cfg1 + cfg2 e2e, A/B
O=gpurun_out/s3o; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_staging.py tests/test_gpu_shapes.py tests/test_gpu_loader.py tests/test_gpu_deflate.py -x -q > $O/pytest_packed.log 2>&1; echo "exit $?" >> $O/pytest_packed.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
RFL_PACK_DELTAS=0 timeout 600 python bench.py --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > $O/bench_cfg1_u8.json 2> $O/bench_cfg1_u8.err
timeout 600 python bench.py --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > $O/bench_cfg1_b.json 2> $O/bench_cfg1_b.err
timeout 1800 python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
