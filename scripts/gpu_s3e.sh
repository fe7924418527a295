#!/bin/bash
# e2e host-time probe (cfg4 / cfg1), cfg4 value with 10 batches per launch, GPU tests
O=gpurun_out/s3e; mkdir -p $O
timeout 600 python scripts/e2e_probe.py cfg4 8 800 > $O/probe_cfg4.txt 2>&1
RFL_TRACE_LOADER=1 timeout 300 python scripts/e2e_probe.py cfg4 8 160 > $O/probe_cfg4_trace.txt 2>&1
timeout 300 python scripts/e2e_probe.py cfg1 1 100 > $O/probe_cfg1.txt 2>&1
timeout 600 python bench.py --workload cfg4 --no-file-e2e --no-verbatim-e2e --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
