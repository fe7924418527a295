#!/bin/bash
# Round-2 evidence pass: GPU tests, smoke, every workload's bench line (+ reference arm), the
# kernel table (graph replay), launch list of the default bench, ncu --set full of the main kernels.
# Usage (repo root, under gpurun): bash scripts/gpu_final_s3.sh [tag]
T=${1:-final}
O=gpurun_out/$T; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1; nproc >> $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
for w in cfg3 cfg4 cfg5; do timeout 1200 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 900 python scripts/kbench.py --graph > $O/kbench.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg1.csv \
   python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-verbatim-e2e --no-file-e2e > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_densify -s 3 -c 1 \
   -o $O/prof_densify_cfg1 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-verbatim-e2e --no-file-e2e > $O/ncu_densify.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_onehot_gather -s 3 -c 1 \
   -o $O/prof_onehot_cfg4 -f python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-verbatim-e2e --no-file-e2e > $O/ncu_onehot.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_gather -s 3 -c 1 \
   -o $O/prof_dense_cfg3 -f python bench.py --workload cfg3 --steps 4 --warmup 3 --no-cpu-baseline --no-verbatim-e2e --no-file-e2e > $O/ncu_dense.log 2>&1
timeout 1800 python bench.py --workload cfg2 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
# (gpurun brings back <= 64 MiB: the reports are summarised here and dropped)
for r in $O/*.ncu-rep; do python scripts/ncu_summary.py $r > ${r%.ncu-rep}.json 2>&1; done
rm -f $O/*.ncu-rep
echo done >> $O/gpu.txt
