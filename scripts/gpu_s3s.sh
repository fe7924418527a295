#!/bin/bash
# host NUMA layout; packed-delta width test; cfg1 e2e repeatability (3 runs)
O=gpurun_out/s3s; mkdir -p $O
lscpu > $O/lscpu.txt 2>&1; ls /sys/devices/system/node/ > $O/nodes.txt 2>&1; nvidia-smi topo -m > $O/topo.txt 2>&1
python -c "import torch;print(torch.cuda.get_device_properties(0))" >> $O/topo.txt 2>&1
cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c >> $O/nodes.txt
timeout 600 python -m pytest tests/test_gpu_staging.py -x -q -k "packed_delta_widths or pull_many" > $O/pytest_new.log 2>&1; echo "exit $?" >> $O/pytest_new.log
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline --no-file-e2e --no-verbatim-e2e > $O/bench_cfg1_$i.json 2>&1; done
