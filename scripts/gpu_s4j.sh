#!/bin/bash
# cfg4 e2e vs the staging pull kernel's shape (piece KB : stages : CTAs), G=16, alternating twice
O=gpurun_out/s4j; mkdir -p $O
for r in 1 2; do for v in 16:4:32 16:8:32 16:4:64 32:4:64 8:8:64 16:8:64; do
  echo "== $v" >> $O/probe_pull.txt
  RFL_PULL=$v timeout 300 python scripts/e2e_probe.py cfg4 16 1600 2>&1 | tail -1 >> $O/probe_pull.txt
done; done
