#!/bin/bash
# K4o by whole rows (RFL_OH=rows) vs plain; parity with it forced; cfg3 default (row-TMA K4)
O=gpurun_out/s3l; mkdir -p $O
RFL_OH=rows timeout 900 python -m pytest tests -m gpu -x -q -k "one_hot or onehot" > $O/pytest_ohrows.log 2>&1; echo "exit $?" >> $O/pytest_ohrows.log
RFL_OH=rows timeout 600 python bench.py --workload cfg4 --no-file-e2e --no-verbatim-e2e --no-cpu-baseline > $O/bench_cfg4_rows.json 2> $O/bench_cfg4_rows.err
timeout 600 python bench.py --workload cfg4 --no-file-e2e --no-verbatim-e2e --no-cpu-baseline > $O/bench_cfg4_plain.json 2> $O/bench_cfg4_plain.err
RFL_OH=rows timeout 600 python bench.py --workload cfg4 --no-file-e2e --no-verbatim-e2e --no-cpu-baseline > $O/bench_cfg4_rows2.json 2> $O/bench_cfg4_rows2.err
timeout 600 python bench.py --workload cfg3 --no-file-e2e > $O/bench_cfg3.json 2> $O/bench_cfg3.err
