# densify tile-buffer sweep: K3 (kbench, raw entry) and K3d (loader, coded image)
mkdir -p gpurun_out
T=${1:-i}
O=gpurun_out/sweep_$T.jsonl
timeout 300 python -m pytest tests/test_gpu_staging.py -x -q -k fused --timeout 300 > gpurun_out/pytest_fused_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused_$T.log
for cfg in "" "v9:256:80:16:2:1" "v9:256:40:16:2:2" "v9:256:48:16:2:2" "v9:256:32:16:3:2" "v9:256:32:8:3:2" "v9:256:24:8:3:2" "v9:256:16:8:3:2"; do
  echo "# RFL_DENSIFY=$cfg" >> $O
  RFL_DENSIFY=$cfg timeout 300 python scripts/kbench.py --graph --cases densify_cfg1,densify_norm_cfg2,densify_bf16_cfg1 >> $O 2>&1
done
for cfg in "" "80:2:1" "48:2:2" "40:2:2" "32:3:2" "24:3:2" "16:3:2" "40:3:1" "64:3:1"; do
  echo "# RFL_DENSIFY_D8=$cfg" >> $O
  RFL_DENSIFY_D8=$cfg timeout 300 python scripts/k3d_probe.py >> $O 2>&1
done
RFL_DENSIFY=v9:256:32:8:3:2 timeout 300 python -m pytest tests/test_gpu_shapes.py -x -q -k "cfg1 or cfg2 or normalize" --timeout 300 > gpurun_out/pytest_nb2_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nb2_$T.log
RFL_DENSIFY_D8=32:3:2 timeout 300 python -m pytest tests/test_gpu_staging.py tests/test_gpu_shapes.py -x -q -k "fused or cfg2" --timeout 300 >> gpurun_out/pytest_nb2_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nb2_$T.log
