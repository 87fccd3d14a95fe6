#!/bin/bash
# FILTER (1) vs PAIR (4) vs BLOCK (2) vs AUTO (0) on the large-alphabet configs
mkdir -p gpurun_out
for w in "c3 4" "c3 8" "c3 16" "c3 64" "c2 2" "c2 4" "c2 8" "c2 16" "c2 64"; do
  for st in 1 4 2 0; do timeout 120 python tools/kcount.py $w 64 0 $st; done
done
