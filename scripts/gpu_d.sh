# dense gather A/B (register vs TMA-pipelined), fused staging tests, kernel table
mkdir -p gpurun_out
T=${1:-d}
timeout 600 python -m pytest tests/test_gpu_staging.py -x -q --timeout 300 > gpurun_out/pytest_staging_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_staging_$T.log
C=dense_bf16_cfg3,dense_bf16_cfg3_g2,dense_raw_cfg4,dense_raw_cfg4_g4
echo "# RFL_DG unset (automatic)" >> gpurun_out/kb_dg_$T.jsonl
timeout 600 python scripts/kbench.py --graph --cases $C >> gpurun_out/kb_dg_$T.jsonl 2>&1
for v in t0 t1 t2 b 4; do
  echo "# RFL_DG=$v" >> gpurun_out/kb_dg_$T.jsonl
  RFL_DG=$v timeout 600 python scripts/kbench.py --graph --cases $C >> gpurun_out/kb_dg_$T.jsonl 2>&1
done
for v in t0 t1 t2; do
  RFL_DG=$v timeout 600 python -m pytest tests/test_gpu_shapes.py -x -q -k "cfg3 or cfg4 or one_hot" --timeout 300 > gpurun_out/pytest_dg_${v}_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dg_${v}_$T.log
done
timeout 600 python scripts/kbench.py --graph > gpurun_out/kbench_$T.jsonl 2>&1
