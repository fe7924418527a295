#!/bin/bash
# final tree check of session 4: GPU tests, smoke, default line, reference arm, launch list
O=gpurun_out/s4g; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg1.csv \
   python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-verbatim-e2e --no-file-e2e > $O/ncu_launch.log 2>&1
