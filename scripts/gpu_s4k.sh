#!/bin/bash
# Python batch wrapping: numpy field read, slotted DeviceBatch, cached ctypes id read-back
O=gpurun_out/s4k; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for G in 8 16; do timeout 300 python scripts/e2e_probe.py cfg4 $G 1600 > $O/probe_cfg4_G$G.txt 2>&1; done
RFL_TRACE_LOADER=1 timeout 300 python scripts/e2e_probe.py cfg4 8 200 > $O/probe_cfg4_trace.txt 2>&1
timeout 900 python bench.py --workload cfg4 --no-file-e2e --no-verbatim-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --workload cfg4 --batches-per-launch 16 --no-file-e2e --no-verbatim-e2e --no-cpu-baseline > $O/bench_cfg4_G16.json 2> $O/bench_cfg4_G16.err
timeout 600 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
