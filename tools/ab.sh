#!/bin/bash
# A/B of two builds of libsmgpu (ab/libsmgpu_A.so vs ab/libsmgpu_B.so), interleaved to cancel drift
for rep in 1 2 3; do
  for v in A B; do
    for w in "c2 16 64" "c2 2 64" "c3 4 64" "c2 256 64"; do
      echo -n "$v "; SMGPU_LIB=$PWD/ab/libsmgpu_$v.so timeout 120 python tools/kcount.py $w | sed 's/plans.*//'
    done
  done
done
