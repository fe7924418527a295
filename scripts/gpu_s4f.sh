#!/bin/bash
# value legs with the graph launch submitted behind a device-side spin (no host launch latency in the region)
O=gpurun_out/s4f; mkdir -p $O
timeout 600 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
for w in cfg4 cfg3; do timeout 900 python bench.py --workload $w --no-file-e2e --no-verbatim-e2e > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 900 python bench.py --workload cfg4 --steps 200 --warmup 10 --no-file-e2e --no-verbatim-e2e --no-cpu-baseline > $O/bench_cfg4_k200.json 2> $O/bench_cfg4_k200.err
