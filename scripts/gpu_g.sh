# N=2 (two ranks sharing the box's GPU) bench lines; ncu --set full of K3d (cfg2 shape)
mkdir -p gpurun_out
T=${1:-g}
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
   bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2_$T.json 2> gpurun_out/bench_n2_$T.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
   bench.py --gpus 2 --workload cfg5 > gpurun_out/bench_cfg5_n2_$T.json 2> gpurun_out/bench_cfg5_n2_$T.err
RIFFLE_PROC_ROWS=500000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_densify_d8 -s 8 -c 1 \
   -o gpurun_out/prof_k3d_cfg2_$T -f python bench.py --workload cfg2 --no-cpu-baseline --no-file-e2e --steps 4 --warmup 3 > gpurun_out/ncu_k3d_$T.log 2>&1
RIFFLE_PROC_ROWS=500000 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_$T.csv \
   python bench.py --workload cfg2 --no-cpu-baseline --no-file-e2e --steps 4 --warmup 3 > /dev/null 2>&1
