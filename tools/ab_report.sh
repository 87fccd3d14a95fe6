#!/bin/bash
# A/B of the reporting path of two builds (tools/report_breakdown.py on c2, dense report), interleaved
for rep in 1 2 3; do
  for v in A B; do
    echo -n "$v "; SMGPU_LIB=$PWD/ab/libsmgpu_$v.so timeout 300 python tools/report_breakdown.py
    echo -n "$v "; SMGPU_LIB=$PWD/ab/libsmgpu_$v.so timeout 300 python tools/dense_report.py | tail -1
  done
done
