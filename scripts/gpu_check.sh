#!/bin/bash
# One GPU-box pass: tests, smoke, bench (N=1 and a 2-rank torchrun sharing the
# box's GPU through a gloo control plane), C++ drop-in parity, HBM calibration,
# kernel micro-benchmarks (CUDA-graph replay), pre-shuffle throughput, launch
# list, ncu --set full captures of the densify kernel (cfg1 bench, cfg2 kbench).
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [tag]
set -u
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
nproc >> gpurun_out/gpu_$TAG.txt; lscpu | grep "Model name" >> gpurun_out/gpu_$TAG.txt; free -g >> gpurun_out/gpu_$TAG.txt
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 300 python scripts/hbm_calib.py > gpurun_out/hbm_$TAG.json 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2>> gpurun_out/bench_$TAG.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
   bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2_$TAG.json 2> gpurun_out/bench_n2_$TAG.err
timeout 900 python scripts/kbench.py --graph > gpurun_out/kbench_$TAG.jsonl 2>&1
timeout 900 python scripts/shuffle_bench.py > gpurun_out/shuffle_$TAG.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
   python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_densify -s 3 -c 1 \
   -o gpurun_out/prof_densify_$TAG -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_densify -s 3 -c 1 \
   -o gpurun_out/prof_densify_cfg2_$TAG -f python scripts/kbench.py --cases densify_norm_cfg2 --steps 2 --warmup 3 > gpurun_out/ncu_full_cfg2_$TAG.log 2>&1
echo done
