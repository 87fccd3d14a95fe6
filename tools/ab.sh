#!/bin/bash
# A/B of two builds of libsmgpu (ab/libsmgpu_A.so vs ab/libsmgpu_B.so), interleaved to cancel drift.
# Workloads: $AB_WORK (";"-separated kcount argument lists) or the default set.
IFS=';' read -ra W <<< "${AB_WORK:-c2 16 64;c2 2 64;c3 4 64;c2 256 64}"
for rep in 1 2 3; do
  for v in A B; do
    for w in "${W[@]}"; do
      echo -n "$v "; SMGPU_LIB=$PWD/ab/libsmgpu_$v.so timeout 120 python tools/kcount.py $w | sed 's/plans.*//'
    done
  done
done
