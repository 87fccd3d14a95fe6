#!/bin/bash
# tuning sweep: CTAs per SM x tile size x stages on c2
set -u
for ctas in 1 2 3; do
  for tile in 8192 16384 32768; do
    for st in 4 8; do
      SMGPU_CTAS_PER_SM=$ctas SMGPU_TILE=$tile SMGPU_STAGES=$st timeout 120 python tools/kbench.py --tag "c$ctas t$tile s$st" --reps 3 --per-m 10
    done
  done
done
