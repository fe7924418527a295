# full GPU tests; cfg2 at 10M cells (fused densify from the HBM-resident coded image);
# cfg3/cfg4 with more batches per launch; ncu of the cfg5 pack kernel inside the bench
mkdir -p gpurun_out
T=${1:-e}
B=/tmp/riffle_bench
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/pytest_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$T.log
timeout 1500 python bench.py --workload cfg2 --no-cpu-baseline --no-file-e2e > gpurun_out/bench_cfg2_$T.json 2> gpurun_out/bench_$T.err
timeout 900 python bench.py --workload cfg4 --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > gpurun_out/bench_cfg4_$T.json 2>> gpurun_out/bench_$T.err
timeout 900 python bench.py --workload cfg4 --no-cpu-baseline --no-file-e2e --no-verbatim-e2e --batches-per-launch 8 > gpurun_out/bench_cfg4_g8_$T.json 2>> gpurun_out/bench_$T.err
rm -rf $B/cfg4*
timeout 900 python bench.py --workload cfg3 --no-cpu-baseline --no-file-e2e --no-verbatim-e2e --batches-per-launch 4 > gpurun_out/bench_cfg3_g4_$T.json 2>> gpurun_out/bench_$T.err
rm -rf $B/cfg3*
timeout 900 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/bench_cfg5_$T.json 2>> gpurun_out/bench_$T.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_copy_tma -s 10 -c 1 \
   -o gpurun_out/prof_pack_cfg5_$T -f python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/ncu_pack_$T.log 2>&1
