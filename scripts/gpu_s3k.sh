#!/bin/bash
# K4 by whole rows through TMA (RFL_DG=row) vs the default dense gathers; parity of the row kernel
O=gpurun_out/s3k; mkdir -p $O
C=dense_bf16_cfg3,dense_bf16_cfg3_g2,dense_raw_cfg4,dense_raw_cfg4_g4
for v in default row b; do
  echo "== $v" >> $O/kb_dense.txt
  if [ $v = default ]; then timeout 300 python scripts/kbench.py --graph --cases $C >> $O/kb_dense.txt 2>&1
  else RFL_DG=$v timeout 300 python scripts/kbench.py --graph --cases $C >> $O/kb_dense.txt 2>&1; fi
done
RFL_DG=row timeout 900 python -m pytest tests -m gpu -x -q -k "dense or cfg3 or cfg4 or bf16 or one_hot" > $O/pytest_dgrow.log 2>&1; echo "exit $?" >> $O/pytest_dgrow.log
RFL_DG=row timeout 600 python bench.py --workload cfg3 --no-file-e2e --no-verbatim-e2e --no-cpu-baseline > $O/bench_cfg3_row.json 2> $O/bench_cfg3_row.err
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
