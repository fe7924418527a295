#!/bin/bash
# densify: two alternating tiles vs one (kbench graph replay, cfg1 / cfg1 bf16 / cfg2 norm); K3d tiles
O=gpurun_out/s3j; mkdir -p $O
C=densify_cfg1,densify_bf16_cfg1,densify_norm_cfg2
for v in default v9:256:80:16:2:1 v9:256:40:16:2:2 v9:256:48:16:2:2 v9:256:32:8:3:2 v9:256:56:16:2:2 v9:256:36:8:3:2; do
  echo "== $v" >> $O/kb_densify.txt
  if [ $v = default ]; then timeout 300 python scripts/kbench.py --graph --cases $C >> $O/kb_densify.txt 2>&1
  else RFL_DENSIFY=$v timeout 300 python scripts/kbench.py --graph --cases $C >> $O/kb_densify.txt 2>&1; fi
done
for v in default 40:2:2 48:2:2 32:3:2; do
  echo "== d8 $v" >> $O/k3d.txt
  if [ $v = default ]; then timeout 600 python scripts/k3d_probe.py >> $O/k3d.txt 2>&1
  else RFL_DENSIFY_D8=$v timeout 600 python scripts/k3d_probe.py >> $O/k3d.txt 2>&1; fi
done
