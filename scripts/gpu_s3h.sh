#!/bin/bash
# evidence pass: launch list of the default bench; ncu --set full of K4o (cfg4 value leg) and of the
# staging pull (cfg1 e2e leg); cfg3 / cfg5 bench lines with the pull staging
O=gpurun_out/s3h; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg1.csv \
   python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-verbatim-e2e --no-file-e2e > $O/ncu_launch_cfg1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_pull -s 6 -c 1 \
   -o $O/prof_pull_cfg1 -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-verbatim-e2e --no-file-e2e > $O/ncu_pull.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_onehot_gather -s 3 -c 1 \
   -o $O/prof_onehot_cfg4 -f python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-verbatim-e2e --no-file-e2e > $O/ncu_onehot.log 2>&1
timeout 900 python bench.py --workload cfg3 --no-file-e2e > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 900 python bench.py --workload cfg5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
