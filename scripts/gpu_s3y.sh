#!/bin/bash
# cfg3 value leg: batches per launch 2 / 4 / 5 / 10 (whole-row TMA gather)
O=gpurun_out/s3y; mkdir -p $O
for g in 2 4 5 10 2 4; do timeout 600 python bench.py --workload cfg3 --batches-per-launch $g --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > $O/bench_cfg3_g$g.json 2>&1; python - "$O/bench_cfg3_g$g.json" $g >> $O/summary.txt <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[2], round(d['value'] / 1e6, 1), round(d['roofline']['frac'], 3), d['roofline']['avg_launch_ms'])
PY
done
