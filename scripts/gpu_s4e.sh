#!/bin/bash
# streamed row-ref loop: non-temporal stores (RFL_REFS_NT=1) vs plain, same box, alternating
O=gpurun_out/s4e; mkdir -p $O
RFL_REFS_NT=1 timeout 900 python -m pytest tests/test_gpu_loader.py tests/test_gpu_shapes.py -m gpu -q -x > $O/pytest_nt.log 2>&1; echo "pytest rc=$?" >> $O/pytest_nt.log
for r in 1 2; do for nt in 0 1; do
  RFL_REFS_NT=$nt timeout 300 python scripts/e2e_probe.py cfg4 8 800 > $O/probe_cfg4_nt${nt}_$r.txt 2>&1
done; done
RFL_REFS_NT=1 RFL_TRACE_LOADER=1 timeout 300 python scripts/e2e_probe.py cfg4 8 200 > $O/probe_cfg4_trace_nt1.txt 2>&1
RFL_TRACE_LOADER=1 timeout 300 python scripts/e2e_probe.py cfg4 8 200 > $O/probe_cfg4_trace_nt0.txt 2>&1
for nt in 0 1; do RFL_REFS_NT=$nt timeout 900 python bench.py --workload cfg4 --steps 200 --warmup 10 --no-file-e2e --no-verbatim-e2e --no-cpu-baseline > $O/bench_cfg4_nt$nt.json 2> $O/bench_cfg4_nt$nt.err; done
for nt in 0 1; do RFL_REFS_NT=$nt timeout 600 python bench.py --no-file-e2e --no-verbatim-e2e --no-cpu-baseline > $O/bench_cfg1_nt$nt.json 2> $O/bench_cfg1_nt$nt.err; done
