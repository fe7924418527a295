#!/bin/bash
# one release event per group (store-owned ring); probes; GPU tests; cfg1 + cfg4 bench
O=gpurun_out/s3g; mkdir -p $O
timeout 600 python scripts/e2e_probe.py cfg4 8 800 > $O/probe_cfg4.txt 2>&1
RFL_TRACE_LOADER=1 timeout 300 python scripts/e2e_probe.py cfg4 8 160 > $O/probe_cfg4_trace.txt 2>&1
timeout 300 python scripts/e2e_probe.py cfg1 1 100 > $O/probe_cfg1.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 300 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 600 python bench.py --workload cfg4 --no-file-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
