#!/bin/bash
# ncu --set full of the cfg3 dense gather at the new default (4 batches per launch)
O=gpurun_out/s4l; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_gather_rows -s 1 -c 1 \
   -o $O/prof_dense_cfg3_g4 -f python bench.py --workload cfg3 --steps 4 --warmup 4 --no-cpu-baseline --no-verbatim-e2e --no-file-e2e > $O/ncu_dense.log 2>&1
for r in $O/*.ncu-rep; do python scripts/ncu_summary.py $r > ${r%.ncu-rep}.json 2>&1; done
rm -f $O/*.ncu-rep
