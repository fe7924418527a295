#!/bin/bash
# staging pull kernel: GPU tests, cfg1 e2e A/B (pull shapes vs copy engine), cfg4 with K4o
O=gpurun_out/s3d; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 300 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
for v in 16:4:32 32:4:32 16:4:64 16:8:32 16:4:16; do RFL_PULL=$v timeout 300 python bench.py --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > $O/bench_cfg1_pull$v.json 2>&1; done
RFL_STAGE=ce timeout 300 python bench.py --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > $O/bench_cfg1_ce.json 2>&1
timeout 600 python bench.py --workload cfg4 --no-file-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
