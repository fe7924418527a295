#!/bin/bash
# fast row->block division in the group loops; K4o bulk-store A/B; GPU tests
O=gpurun_out/s3f; mkdir -p $O
timeout 600 python scripts/e2e_probe.py cfg4 8 800 > $O/probe_cfg4.txt 2>&1
RFL_TRACE_LOADER=1 timeout 300 python scripts/e2e_probe.py cfg4 8 160 > $O/probe_cfg4_trace.txt 2>&1
timeout 300 python scripts/e2e_probe.py cfg1 1 100 > $O/probe_cfg1.txt 2>&1
timeout 600 python bench.py --workload cfg4 --no-file-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
RFL_OH=bulk timeout 600 python bench.py --workload cfg4 --no-file-e2e --no-verbatim-e2e --no-cpu-baseline > $O/bench_cfg4_ohbulk.json 2> $O/bench_cfg4_ohbulk.err
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
RFL_OH=bulk timeout 600 python -m pytest tests -m gpu -x -q -k "one_hot or onehot" > $O/pytest_ohbulk.log 2>&1
