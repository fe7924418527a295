#!/bin/bash
# final check of the committed tree: GPU tests, smoke, default bench line, reference arm
O=gpurun_out/s3w; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py --workload cfg4 --steps 200 --warmup 10 --no-file-e2e > $O/bench_cfg4_k200.json 2> $O/bench_cfg4_k200.err
