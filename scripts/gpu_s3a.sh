#!/bin/bash
# round-2 session-3 pass: PCIe lanes calibration, GPU tests, default bench line, reference arm, smoke
O=gpurun_out/s3a; mkdir -p $O
nvidia-smi -L > $O/gpu.txt
timeout 120 scripts/cuda/h2d_pattern > $O/h2d_lanes.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
for L in 1 2 4; do RFL_COPY_LANES=$L timeout 300 python bench.py --no-cpu-baseline --no-file-e2e > $O/bench_cfg1_lanes$L.json 2> $O/bench_cfg1_lanes$L.err; done
timeout 300 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 300 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
