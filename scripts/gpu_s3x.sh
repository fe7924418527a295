#!/bin/bash
# stream_file through the staging pull: parity (every stream_file / deflate / shape test), e2e A/B
O=gpurun_out/s3x; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for i in 1 2; do
RIFFLE_E2E_STAGING=stream_file timeout 300 python bench.py --no-cpu-baseline --no-verbatim-e2e --no-file-e2e > $O/bench_file_pull_$i.json 2>&1
RFL_STAGE=ce RIFFLE_E2E_STAGING=stream_file timeout 300 python bench.py --no-cpu-baseline --no-verbatim-e2e --no-file-e2e > $O/bench_file_ce_$i.json 2>&1
done
