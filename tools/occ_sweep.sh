#!/bin/bash
# occupancy knobs (CTAs per SM x tile bytes) on the slowest large-alphabet cases and the c2 step
mkdir -p gpurun_out
for cfg in "2 32768" "3 16384" "4 16384" "3 8192" "4 8192"; do
  set -- $cfg
  echo "== ctas=$1 tile=$2"
  for w in "c3 4" "c3 8" "c3 16" "c2 2" "c2 4" "c2 16"; do
    SMGPU_CTAS_PER_SM=$1 SMGPU_TILE=$2 timeout 120 python tools/kcount.py $w 64
  done
done
