#!/bin/bash
# K4o tiled (default) vs plain; cfg5 with the pack / D2H gate on / off; GPU tests touching them
O=gpurun_out/s3i; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "one_hot or onehot or shuffle or preshuffle" > $O/pytest_sel.log 2>&1; echo "exit $?" >> $O/pytest_sel.log
timeout 600 python bench.py --workload cfg4 --no-file-e2e --no-verbatim-e2e --no-cpu-baseline > $O/bench_cfg4_tile.json 2> $O/bench_cfg4_tile.err
RFL_OH=plain timeout 600 python bench.py --workload cfg4 --no-file-e2e --no-verbatim-e2e --no-cpu-baseline > $O/bench_cfg4_plain.json 2> $O/bench_cfg4_plain.err
timeout 900 python bench.py --workload cfg5 --no-cpu-baseline > $O/bench_cfg5_gate.json 2> $O/bench_cfg5_gate.err
RFL_PACK_GATE=0 timeout 900 python bench.py --workload cfg5 --no-cpu-baseline > $O/bench_cfg5_nogate.json 2> $O/bench_cfg5_nogate.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_onehot_gather -s 3 -c 1 \
   -o $O/prof_onehot_tile_cfg4 -f python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-verbatim-e2e --no-file-e2e > $O/ncu_onehot.log 2>&1
