mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tile_sweep scripts/cuda/tile_sweep.cu > /dev/null 2>&1
timeout 600 /tmp/tile_sweep > gpurun_out/tile_sweep_h.jsonl 2>&1
