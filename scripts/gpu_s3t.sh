#!/bin/bash
# write-only HBM ceilings (mix_bw); staging tests after the NUMA placement change
O=gpurun_out/s3t; mkdir -p $O
timeout 300 scripts/cuda/mix_bw > $O/mix_bw.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_staging.py tests/test_gpu_loader.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > $O/bench_cfg1.json 2>&1
