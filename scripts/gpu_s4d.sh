#!/bin/bash
# session-4 evidence pass (scripts/gpu_final_s3.sh) + cfg3 batches-per-launch A/B
bash scripts/gpu_final_s3.sh final_s4
O=gpurun_out/final_s4
for g in 4 5; do timeout 600 python bench.py --workload cfg3 --batches-per-launch $g --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > $O/bench_cfg3_g$g.json 2> $O/bench_cfg3_g$g.err; done
