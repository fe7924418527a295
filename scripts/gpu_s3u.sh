#!/bin/bash
# K4o: groups of rows per 16 KB bulk store (RFL_OH=rows4) vs one row per store; parity
O=gpurun_out/s3u; mkdir -p $O
C=onehot_cfg4,onehot_cfg4_g10,onehot_bf16_cfg4_g4
for v in default rows4 plain default rows4; do
  echo "== $v" >> $O/kb_onehot.txt
  if [ $v = default ]; then timeout 300 python scripts/kbench.py --graph --cases $C >> $O/kb_onehot.txt 2>&1
  else RFL_OH=$v timeout 300 python scripts/kbench.py --graph --cases $C >> $O/kb_onehot.txt 2>&1; fi
done
RFL_OH=rows4 timeout 900 python -m pytest tests -m gpu -x -q -k "one_hot or onehot" > $O/pytest_rows4.log 2>&1; echo "exit $?" >> $O/pytest_rows4.log
