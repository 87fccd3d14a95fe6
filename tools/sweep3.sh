#!/bin/bash
set -u
for cfg in "2 16384" "2 32768" "1 32768" "3 16384"; do
  set -- $cfg
  SMGPU_CTAS_PER_SM=$1 SMGPU_TILE=$2 timeout 120 python tools/kbench.py --tag "c$1 t$2" --reps 3 --per-m 10 --lengths 2,4,8,16,64,256,1024
done
