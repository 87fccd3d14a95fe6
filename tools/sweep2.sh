#!/bin/bash
set -u
for ctas in 1 2; do
  for tile in 8192 16384 32768; do
    SMGPU_CTAS_PER_SM=$ctas SMGPU_TILE=$tile timeout 120 python tools/kbench.py --tag "c$ctas t$tile" --reps 3 --per-m 10 --lengths 2,4,8,16,64,256,1024
  done
done
