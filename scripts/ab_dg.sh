#!/bin/bash
# dense gather unit sweep (RFL_DG=2|4 loads per lane; the session-3 sweep also had 1/3/6/8 and
# 128/512-thread CTAs, profiles/r1_dense_gather.md) + filesystem write calibration
mkdir -p gpurun_out
T=${1:-s3e}
for s in 2 4; do
  echo "== $s" >> gpurun_out/kb_${T}_dg.txt
  RFL_DG=$s timeout 300 python scripts/kbench.py --graph --cases dense_bf16_cfg3,dense_raw_cfg4 >> gpurun_out/kb_${T}_dg.txt 2>&1
done
{ df -h /tmp; mount | grep -E " /tmp | / "; nproc; free -g;
  dd if=/dev/zero of=/tmp/ddtest bs=64M count=64 2>&1 | tail -1;
  dd if=/dev/zero of=/tmp/ddtest bs=64M count=64 conv=fdatasync 2>&1 | tail -1; rm -f /tmp/ddtest;
  dd if=/dev/zero of=/dev/shm/ddtest bs=64M count=64 2>&1 | tail -1; rm -f /dev/shm/ddtest; df -h /dev/shm; } > gpurun_out/fs_$T.txt 2>&1
echo done
