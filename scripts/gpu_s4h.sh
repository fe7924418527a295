#!/bin/bash
# cfg4 e2e: batches per C call / launch 8 vs 16 vs 32 (same box)
O=gpurun_out/s4h; mkdir -p $O
for G in 8 16 32 8 16 32; do
  timeout 300 python scripts/e2e_probe.py cfg4 $G 1600 >> $O/probe_cfg4_G$G.txt 2>&1
done
for G in 8 16; do timeout 900 python bench.py --workload cfg4 --batches-per-launch $G --no-file-e2e --no-verbatim-e2e --no-cpu-baseline > $O/bench_cfg4_G$G.json 2> $O/bench_cfg4_G$G.err; done
