#!/bin/bash
# stream_file e2e: where the time goes (cfg1), read-ahead depth sweep
O=gpurun_out/s3r; mkdir -p $O
RIFFLE_E2E_STAGING=stream_file timeout 300 python scripts/e2e_probe.py cfg1 1 60 > $O/probe_file.txt 2>&1
RIFFLE_E2E_STAGING=stream_file RFL_TRACE_LOADER=1 timeout 300 python scripts/e2e_probe.py cfg1 1 30 > $O/probe_file_trace.txt 2>&1
for d in 4 8 16; do RIFFLE_E2E_DEPTH=$d RIFFLE_E2E_STAGING=stream_file timeout 300 python bench.py --no-cpu-baseline --no-verbatim-e2e --no-file-e2e > $O/bench_file_d$d.json 2>&1; done
nproc > $O/host.txt; free -g >> $O/host.txt; df -h /tmp >> $O/host.txt
