#!/bin/bash
# group bases in the resident_coded image: parity, K3d A/B, cfg2 line
O=gpurun_out/s3v; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_staging.py tests/test_gpu_shapes.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for v in 1 0 1 0; do echo "== bases $v" >> $O/k3d.txt; RFL_GROUP_BASES=$v timeout 600 python scripts/k3d_probe.py >> $O/k3d.txt 2>&1; done
timeout 1800 python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
