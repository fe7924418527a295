#!/bin/bash
# round-2 session 4b: per-block live-row counts from the replay thread, ids D2H through rfl_ids_download_async
O=gpurun_out/s4b; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python scripts/e2e_probe.py cfg4 8 800 > $O/probe_cfg4.txt 2>&1
RFL_TRACE_LOADER=1 timeout 300 python scripts/e2e_probe.py cfg4 8 200 > $O/probe_cfg4_trace.txt 2>&1
timeout 300 python scripts/e2e_probe.py cfg1 1 100 > $O/probe_cfg1.txt 2>&1
timeout 900 python bench.py --workload cfg4 --steps 200 --warmup 10 --no-file-e2e > $O/bench_cfg4_k200.json 2> $O/bench_cfg4_k200.err
timeout 600 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > $O/smoke.log 2>&1
