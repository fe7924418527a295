#!/bin/bash
mkdir -p gpurun_out
T=${1:-s3l}
export RIFFLE_BENCH_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
   bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2_$T.json 2> gpurun_out/bench_n2_$T.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
   bench.py --gpus 2 --workload cfg5 > gpurun_out/bench_cfg5_n2_$T.json 2> gpurun_out/bench_cfg5_n2_$T.err
unset RIFFLE_BENCH_BACKEND
rm -rf /tmp/riffle_bench/cfg5*
sync; echo 3 > /proc/sys/vm/drop_caches 2>/dev/null
for d in 4 16; do RIFFLE_E2E_STAGING=stream_file RIFFLE_E2E_DEPTH=$d timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_sf${d}_$T.json 2>&1; done
KB_SCHED=1 timeout 600 python scripts/kbench.py --graph --cases dense_bf16_cfg3,dense_raw_cfg4,densify_cfg1 > gpurun_out/kb_${T}_sched.jsonl 2>&1
echo done
